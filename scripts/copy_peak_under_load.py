"""Is the HBM roofline itself clock-dependent? Time the driver's peak recipe (b.copy_(a) over
1 Gi bf16, read+write bytes) clean and right after a bf16 GEMM burst (power-capped SM clocks),
next to fused_adamw_pack under the same two conditions."""
import json
import os
import statistics
import sys
import subprocess

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

dev = torch.device("cuda", 0)
a = torch.empty(1 << 30, dtype=torch.bfloat16, device=dev)
b = torch.empty_like(a)
A = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
B = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)


def clocks():
    try:
        out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits"],
                             capture_output=True, text=True).stdout.strip()
        return float(out.splitlines()[0])
    except Exception:
        return None


res = {}
for burst in (False, True):
    ts = []
    for _ in range(12):
        if burst:
            for _ in range(8):
                torch.mm(A, B)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        b.copy_(a)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    res["copy_gemm" if burst else "copy_clean"] = {"best_gbs": 2 * 2 * (1 << 30) / min(ts[2:]) / 1e6,
                                                   "median_gbs": 2 * 2 * (1 << 30) / statistics.median(ts[2:]) / 1e6,
                                                   "sm_mhz_after": clocks()}
print(json.dumps(res))
