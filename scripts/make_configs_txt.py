"""Summarise the round-2 config bench lines (scripts/gpu_r02_configs.sh) into one table (CPU).

python scripts/make_configs_txt.py gpurun_out/cfg profiles/r02_configs.txt
"""
import json
import os
import statistics
import sys

src, dst = sys.argv[1], sys.argv[2]
rows = []
for f in sorted(os.listdir(src)):
    if not f.endswith(".json"):
        continue
    name = f[:-5]
    try:
        lines = [json.loads(l) for l in open(os.path.join(src, f)) if l.startswith("{")]
    except Exception:
        lines = []
    if not lines:
        err = open(os.path.join(src, name + ".err")).read()[-300:] if os.path.exists(os.path.join(src, name + ".err")) else ""
        rows.append((name, None, err.strip().splitlines()[-1] if err.strip() else "no output"))
        continue
    d = lines[-1]
    steps = []
    sp = os.path.join(src, name + ".steps.jsonl")
    if os.path.exists(sp):
        steps = [json.loads(l) for l in open(sp)]
    rows.append((name, d, steps))

out = ["Round-2 BASELINE config lines (one B200; bench.py, default = ring staging, host batch replay, drain",
       "verification on). stall = mean step-time increase of a session step over the checkpoint-free median",
       "of the same run; per-ckpt = stall x K; wait = event-timed slot/state wait per session step; thr = throughput",
       "with checkpointing / checkpoint-free; kernel = fused AdamW(+pack) plain-launch HBM fraction (live, vs the",
       "pod's measured copy peak); replay = host replay arithmetic of the last session; steps = per-step JSONL rows.",
       "",
       f"{'config':28s} {'n_per_rank':>13s} {'K':>3s} {'I':>4s} {'stall ms':>9s} {'% step':>7s} {'per-ckpt':>9s} "
       f"{'wait ms':>8s} {'thr':>7s} {'D2H GB/s':>9s} {'link':>6s} {'kernel':>7s} {'replay ms':>10s} {'SM MHz':>7s} "
       f"{'steps':>6s}"]
for name, d, steps in rows:
    if d is None:
        out.append(f"{name:28s} FAILED: {steps}")
        continue
    st, c = d["stall"], d["config"]
    K = c["K"]
    out.append(f"{name:28s} {c['n_per_rank']:13,d} {K:3d} {c['interval']:4d} {st['delta_ms_per_session_step_mean']:9.3f} "
               f"{100 * st['delta_frac_of_step']:6.2f}% {st['delta_ms_per_session_step_mean'] * K:9.2f} "
               f"{st['wait_ms_per_session_step']:8.3f} {d['ckpt_free']['throughput_ratio']:7.4f} "
               f"{(d['d2h']['gbs'] or 0):9.1f} {d['d2h']['link_peak_gbs']:6.1f} {100 * d['roofline']['frac']:6.1f}% "
               f"{d['replay']['host_ms_last_session']:10.1f} {str((d.get('clocks') or {}).get('sm_mhz')):>7s} {len(steps):6d}")
out.append("")
for name, d, steps in rows:
    if d is None or not steps:
        continue
    sess = [s for s in steps if s["part"]]
    if not sess:
        continue
    out.append(f"{name}: {len(sess)} session steps logged; median t_step {statistics.median(s['t_step_ms'] for s in sess):.2f} ms, "
               f"max wait {max(s['wait_ms'] for s in sess):.3f} ms, median fused {statistics.median(s['fused_ms'] for s in sess):.3f} ms, "
               f"D2H per step {statistics.median(s['d2h_bytes'] for s in sess) / 1e9:.2f} GB in "
               f"{statistics.median(s['d2h_ms'] for s in sess):.1f} ms")
open(dst, "w").write("\n".join(out) + "\n")
print("\n".join(out))
