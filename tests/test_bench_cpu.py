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


def test_reference_arm_other_ranks_exit_quietly():
    out = run(["--impl", "reference", "--steps", "1", "--warmup", "1", "--cpu-sample", str(1 << 16)],
              env={"WORLD_SIZE": "2", "RANK": "1", "LOCAL_RANK": "1"})
    assert out.strip() == ""


def test_resolve_shards():
    sys.path.insert(0, ROOT)
    import importlib
    bench = importlib.import_module("bench")
    for model, W, want in [("gpt2-small", 1, 124_439_808), ("llama2-7b", 8, 842_301_952),
                           ("llama2-13b", 8, 1_626_983_424)]:
        a = type("A", (), dict(model=model, shard_of=W, n=0, tokens=0))()
        bench.resolve(a)
        assert a.n == want and a.tokens > 0 and a.W == W
