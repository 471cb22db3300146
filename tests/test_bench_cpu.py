"""bench.py's CPU-side contract (-m "not gpu"): the reference arm (the oracle timed on host cores)
prints one JSON line with the contract's keys, and exits 0 without work on ranks != 0."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(args, env=None):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=600, env=dict(os.environ, **(env or {})))
    assert r.returncode == 0, r.stderr
    return r.stdout


def test_reference_arm_json_line():
    out = run(["--impl", "reference", "--steps", "2", "--warmup", "1", "--cpu-sample", str(1 << 18),
               "--interval", "10", "--K", "4"])
    lines = [l for l in out.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "tokens/s"
    assert d["config"]["workload"].startswith("GPT-2 small")
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    cb = d["cpu_baseline"]
    assert cb["sample_elements"] == 1 << 18 and cb["samples_timed"] == 2
    assert abs(cb["measured_s_per_interval_sample"] * cb["extrapolation_factor"] - cb["extrapolated_s_per_interval"]) < 1e-9


def test_reference_arm_other_ranks_exit_quietly():
    out = run(["--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "1", "--cpu-sample", str(1 << 16)],
              env={"WORLD_SIZE": "2", "RANK": "1", "LOCAL_RANK": "1"})
    assert out.strip() == ""


def test_gpus_must_match_world_size():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "4"],
                       capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0"))
    assert r.returncode != 0 and "WORLD_SIZE=2" in r.stderr


def test_gpus_n_without_torchrun_relaunches_itself():
    """`python bench.py --gpus 2` with no torchrun environment re-executes under
    torch.distributed.run (2 local ranks over gloo here) and prints exactly one line, n_gpus == 2."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR",
                                                             "MASTER_PORT")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--dist-backend", "gloo", "--steps", "1", "--warmup", "0", "--cpu-sample", str(1 << 16),
                        "--interval", "6", "--K", "2"],
                       capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2 and lines[0]["impl"] == "reference"


def test_reference_and_gpu_arm_share_the_config():
    """The driver pairs the two arms by config: both lines build it with config_dict (the GPU arm
    only overrides K with the K it used, equal to --K unless --K 0)."""
    sys.path.insert(0, ROOT)
    import importlib
    bench = importlib.import_module("bench")
    a = type("A", (), dict(model="gpt2-small", shard_of=0, n=0, tokens=0, K=8, interval=50, copy_mode="ce",
                           ring_slots=2, staging="ring", scheme="gockpt", replay_mode="host",
                           dist_backend="nccl", rs_bucket_mb=512, spin_ms=1.0, verify_drain=1, plan="equal"))()
    bench.resolve(a)
    c1 = bench.config_dict(a, 1)
    assert dict(c1, K=8) == c1 and c1["fb_tflop_per_step"] > 10 and c1["n_per_rank"] == 124_439_808
    assert c1["plan"] == "equal"                                   # the partition plan is part of the workload key


def test_resolve_shards():
    sys.path.insert(0, ROOT)
    import importlib
    bench = importlib.import_module("bench")
    for model, W, want in [("gpt2-small", 1, 124_439_808), ("llama2-7b", 8, 842_301_952),
                           ("llama2-13b", 8, 1_626_983_424)]:
        a = type("A", (), dict(model=model, shard_of=W, n=0, tokens=0))()
        bench.resolve(a)
        assert a.n == want and a.tokens > 0 and a.W == W


def test_rs_buckets_cover_the_shard():
    """The ZeRO-1 reduce-scatter buckets (N > 1 with NCCL): contiguous, in order, covering [0, n) of the
    rank's shard, each input (world x count bf16) at most the bucket size, counts 512-aligned but the last."""
    sys.path.insert(0, ROOT)
    from paper_2511_07035_b200.harness import rs_buckets
    for n, world, mb in [(842_301_952, 8, 512), (3_253_966_336, 4, 512), (124_439_808, 2, 64), (1000, 8, 512)]:
        b = rs_buckets(n, world, mb << 20)
        assert b[0][0] == 0 and sum(c for _, c in b) == n
        assert all(o2 == o1 + c1 for (o1, c1), (o2, _) in zip(b, b[1:]))
        assert all(2 * world * c <= max(mb << 20, 2 * world * 512) for _, c in b)
        assert all(c % 512 == 0 for _, c in b[:-1])


def test_standin_flops_match_the_model_shapes():
    """The stand-in's analytic FLOPs (config fb_tflop_per_step, both arms) = 3 x 2 MKN over its GEMMs;
    ~6 x params x tokens for the matmul weights plus attention."""
    sys.path.insert(0, ROOT)
    from paper_2511_07035_b200.harness import MODELS, standin_flops
    for model, tokens in [("gpt2-small", 16384), ("llama2-7b", 8192), ("llama2-13b", 2048)]:
        f = standin_flops(model, tokens)
        params = MODELS[model][0]
        assert 5.5 * params * tokens < f < 9.0 * params * tokens, (model, f / (params * tokens))
