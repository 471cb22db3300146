"""Ceiling of an all-bulk-copy (TMA load + TMA store) version of the fused kernel's 8-stream pattern
(28 B/element, no arithmetic), next to the LDG/STG grid-stride copy (stream8.cu) and torch's copy.
Decides whether moving the fused kernel's stores to bulk S2G can raise its HBM fraction."""
import ctypes as C
import json
import os
import statistics
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

here = os.path.dirname(os.path.abspath(__file__))
libs = {}
for name in ("stream8", "stream8_tma"):
    so = f"/tmp/lib{name}.so"
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler", "-fPIC",
                    os.path.join(here, "cuda", f"{name}.cu"), "-o", so], check=True)
    libs[name] = C.CDLL(so)
n = 124_439_808
p = torch.zeros(n, device="cuda")
m, v = torch.zeros_like(p), torch.zeros_like(p)
g = torch.randint(-32768, 32767, (n,), dtype=torch.int16, device="cuda")
out = torch.zeros_like(g)
args = [C.c_void_p(t.data_ptr()) for t in (p, m, v, g, out)]
sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)


GEMM = os.environ.get("GCK_MB_GEMM") == "1"   # a GEMM burst before each launch (power-capped clocks)
if GEMM:
    A = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
    Bm = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)


def timeit(fn, iters=30):
    ts = []
    for it in range(iters):
        if GEMM:
            for _ in range(8):
                torch.mm(A, Bm)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        rc = fn()
        b.record()
        torch.cuda.synchronize()
        assert rc == 0, rc
        if it >= 5:
            ts.append(a.elapsed_time(b))
    return {"us_mean": statistics.mean(ts) * 1e3, "gbs": 28 * n / (statistics.mean(ts) / 1e3) / 1e9,
            "gbs_best": 28 * n / (min(ts) / 1e3) / 1e9}


res = {}
for blocks in (148 * 4, 148 * 8):
    res[f"ldg_stg_{blocks}blk"] = timeit(lambda: libs["stream8"].run_stream8(*args, C.c_uint64(n), blocks, sp))
cfgs = {0: ("4st x 2048, lag1", 148, 2048), 1: ("6st x 2048, lag2", 148, 2048), 2: ("7st x 2048, lag3", 148, 2048),
        3: ("3st x 4096, lag1", 148, 4096), 4: ("3st x 2048, lag1, 2 CTA/SM", 296, 2048)}
for cfg, (label, blocks, tile) in cfgs.items():
    out.zero_()
    res[f"tma_{label}"] = timeit(lambda: libs["stream8_tma"].run_tma8(*args, C.c_uint64(n), blocks, cfg, sp))
    tiles = n // tile * tile
    res[f"tma_{label}"]["bytes_ok"] = bool(torch.equal(out[:tiles], g[:tiles]))
x = torch.empty(1 << 30, dtype=torch.bfloat16, device="cuda")
y = torch.empty_like(x)
ts = []
for it in range(15):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    y.copy_(x)
    b.record()
    torch.cuda.synchronize()
    if it >= 3:
        ts.append(a.elapsed_time(b))
res["torch_copy_1Gi_bf16"] = {"gbs": 4 * (1 << 30) / (statistics.mean(ts) / 1e3) / 1e9}
res["gemm_burst"] = GEMM
print(json.dumps(res, indent=1))
