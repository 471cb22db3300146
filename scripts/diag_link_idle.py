"""Diagnostic: does an idle host link make the next small D2H copy slow? Times one 4 MiB
device->pinned copy after host idle gaps of 0 / 0.2 / 1 / 5 / 20 ms (CUDA events on the copy's
stream), and reports the PCIe link generation nvidia-smi sees at idle and under a copy loop."""
import json
import subprocess
import time

import torch


def smi():
    try:
        return subprocess.run(["nvidia-smi", "--query-gpu=pcie.link.gen.current,pcie.link.width.current,clocks.sm,clocks.mem",
                               "--format=csv,noheader"], capture_output=True, text=True, timeout=20).stdout.strip()
    except Exception as e:  # noqa: BLE001
        return str(e)


def main():
    torch.cuda.set_device(0)
    d = torch.empty(4 << 20, dtype=torch.uint8, device="cuda")
    h = torch.empty(4 << 20, dtype=torch.uint8, pin_memory=True)
    s = torch.cuda.Stream()
    out = {"idle_smi": smi()}
    for gap_ms in (0, 0.2, 1, 5, 20):
        ts = []
        for r in range(12):
            if gap_ms:
                time.sleep(gap_ms / 1e3)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(s):
                e0.record(s)
                h.copy_(d, non_blocking=True)
                e1.record(s)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts = sorted(ts[2:])
        out[f"gap_{gap_ms}ms"] = {"median_us": ts[len(ts) // 2] * 1e3, "min_us": ts[0] * 1e3, "max_us": ts[-1] * 1e3}
    # a 4 MiB copy with the GPU kept busy by a compute kernel on another stream (the link idle before)
    a = torch.randn(4096, 4096, device="cuda", dtype=torch.bfloat16)
    ts = []
    for r in range(12):
        time.sleep(0.005)
        for _ in range(4):
            a @ a
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            h.copy_(d, non_blocking=True)
            e1.record(s)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts = sorted(ts[2:])
    out["gap_5ms_gemm_busy"] = {"median_us": ts[len(ts) // 2] * 1e3, "min_us": ts[0] * 1e3, "max_us": ts[-1] * 1e3}
    # two copies back to back after an idle gap: is only the first one slow?
    ts1, ts2 = [], []
    for r in range(12):
        time.sleep(0.005)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        with torch.cuda.stream(s):
            ev[0].record(s)
            h.copy_(d, non_blocking=True)
            ev[1].record(s)
            h.copy_(d, non_blocking=True)
            ev[2].record(s)
        ev[2].synchronize()
        ts1.append(ev[0].elapsed_time(ev[1]))
        ts2.append(ev[1].elapsed_time(ev[2]))
    out["gap_5ms_first_second_us"] = [sorted(ts1)[6] * 1e3, sorted(ts2)[6] * 1e3]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
