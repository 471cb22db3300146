"""The N>1 bench path end to end on one GPU (-m gpu): torchrun with 2 ranks sharing the device over
gloo (NCCL refuses two ranks on one GPU; the harness's NCCL collectives are skipped), so per-rank
ZeRO-1 shards, barrier-bracketed timing with the max over ranks, rank-0-only output and the
reference arm's rank handling are exercised as the driver's scaling run would."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def torchrun(args, timeout=900):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"), *args]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    return [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]


def test_two_rank_bench_line():
    lines = torchrun(["--gpus", "2", "--dist-backend", "gloo", "--steps", "2", "--warmup", "3", "--interval", "12",
                      "--no-e2e"])
    assert len(lines) == 1
    d = lines[0]
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["scaling"] == "weak"
    assert d["config"]["n_per_rank"] == (124_439_808 + 2 * 512 - 1) // (2 * 512) * 512
    assert d["gpu_launches"] > 0 and d["roofline"]["achieved"] > 0


def test_two_rank_reference_arm():
    lines = torchrun(["--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "1", "--cpu-sample",
                      str(1 << 18)])
    assert len(lines) == 1 and lines[0]["impl"] == "reference" and lines[0]["value"] > 0


@pytest.mark.parametrize("staging", ["ring", "direct"])
def test_one_gpu_bench_line_with_e2e(staging):
    """The default N=1 launch on a reduced shard, e2e leg included: the gradient is prefetched from
    pinned host memory into alternating device buffers on a copy stream (ring: packed by the fused
    kernel; direct: copied out of the caller's buffer behind gck_grad_fence)."""
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "2", "--warmup", "3", "--interval", "10",
           "--K", "4", "--n", str(1 << 24), "--staging", staging, "--no-cpu-baseline"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = lines[0]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == 2 * (1 << 24) and e["d2h_bytes_per_step"] > 8
    assert d["stall"]["session_steps_measured"] == 2 * 4 and d["gpu_launches"] > 0


def test_gpus_2_without_torchrun_relaunches():
    """`python bench.py --gpus 2` exactly as a user types it (no torchrun environment): bench.py
    re-executes itself under torch.distributed.run; one line, n_gpus == 2, per-rank lists of 2."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dist-backend", "gloo", "--steps", "2",
           "--warmup", "3", "--interval", "12", "--no-e2e"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = lines[0]
    assert d["n_gpus"] == 2 and len(d["per_rank"]["ranks"]) == 2
    assert d["d2h"]["link_peak_alone_gbs"] > 0 and d["d2h"]["link_peak_concurrent_gbs"] > 0


def test_flat_1m_line_and_step_log(tmp_path):
    """BASELINE config 1 as a bench line (F/B = a 1 ms spin kernel) with the per-step JSONL log."""
    log = tmp_path / "steps.jsonl"
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--model", "flat-1m", "--K", "4", "--interval", "10",
           "--steps", "3", "--warmup", "3", "--spin-ms", "1", "--step-log", str(log), "--no-cpu-baseline"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    d = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")][0]
    assert d["unit"] == "steps/s" and d["config"]["n_per_rank"] == 1 << 20 and d["config"]["K"] == 4
    assert d["config"]["workload"].startswith("flat 1M")
    recs = [json.loads(l) for l in open(log)]
    assert len(recs) == 3 * 10 - 1
    assert [r_["part"] for r_ in recs[:10]] == [1, 2, 3, 4, 0, 0, 0, 0, 0, 0]
    sess = [r_ for r_ in recs if r_["part"]]
    assert all(r_["d2h_bytes"] > 0 and r_["fused_ms"] > 0 and r_["slot"] in (0, 1) for r_ in sess)
    assert sum(r_["d2h_bytes"] for r_ in recs[:10]) == d["d2h"]["bytes_per_session"]


def test_nccl_bucketed_reduce_scatter_path_on_one_gpu():
    """The N > 1 NCCL path of the harness (per-bucket async reduce-scatter during the split backward,
    the param all-gather, NCCL init with INFO lines on stderr) as a process group of one: the only
    NCCL run a one-GPU box allows (NCCL refuses two ranks on one device)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1", "--master-addr",
           "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"), "--gpus", "1",
           "--force-collectives", "--rs-bucket-mb", "64", "--steps", "2", "--warmup", "3", "--interval", "10",
           "--K", "4", "--no-e2e", "--no-cpu-baseline"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    d = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")][0]
    assert d["config"]["rs_bucket_mb"] == 64 and d["value"] > 0 and d["stall"]["session_steps_measured"] == 8
    assert "NCCL INFO" in r.stderr + r.stdout, (r.stderr[-2000:], r.stdout[-2000:])
