"""Achievable HBM bandwidth for the fused kernel's 8-stream access pattern (28 B/element) with no
arithmetic, vs torch's copy (the MEASURED_PEAKS recipe) — the practical ceiling for fused_adamw_pack."""
import ctypes as C
import json
import os
import statistics
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

here = os.path.dirname(os.path.abspath(__file__))
so = "/tmp/libstream8.so"
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler", "-fPIC",
                os.path.join(here, "cuda", "stream8.cu"), "-o", so], check=True)
L = C.CDLL(so)
n = 124_439_808
p = torch.zeros(n, device="cuda")
m, v = torch.zeros_like(p), torch.zeros_like(p)
g = torch.zeros(n, dtype=torch.int16, device="cuda")
out = torch.zeros_like(g)
res = {}
for blocks in (148 * 2, 148 * 4, 148 * 8):
    ts = []
    for it in range(25):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        L.run_stream8(C.c_void_p(p.data_ptr()), C.c_void_p(m.data_ptr()), C.c_void_p(v.data_ptr()),
                      C.c_void_p(g.data_ptr()), C.c_void_p(out.data_ptr()), C.c_uint64(n), blocks,
                      C.c_void_p(torch.cuda.current_stream().cuda_stream))
        b.record()
        torch.cuda.synchronize()
        if it >= 5:
            ts.append(a.elapsed_time(b))
    res[f"stream8_{blocks}blk"] = {"us_mean": statistics.mean(ts) * 1e3, "gbs": 28 * n / (statistics.mean(ts) / 1e3) / 1e9,
                                   "gbs_best": 28 * n / (min(ts) / 1e3) / 1e9}
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
res["torch_copy_1Gi_bf16"] = {"gbs": 4 * (1 << 30) / (statistics.mean(ts) / 1e3) / 1e9,
                              "gbs_best": 4 * (1 << 30) / (min(ts) / 1e3) / 1e9}
print(json.dumps(res))
