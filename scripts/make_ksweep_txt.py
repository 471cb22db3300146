"""Regenerate profiles/<tag>_k_sweep_and_schemes.txt from the raw K-sweep / 7B / scheme lines."""
import json
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
P = "profiles/"
rows = [json.loads(l) for l in open(P + f"{tag}_k_sweep_llama13b_r8.jsonl") if l.startswith("{")]
lines = ["BASELINE config 4: K sweep on one B200 emulating one rank of an 8-GPU Llama-2 13B ZeRO-1 job",
         "(n_r = 1,626,983,424 fp32 elements; 1x2048 tokens per step -> ~155 ms steps; interval K+8; 2 timed intervals).",
         "stall = mean step-time increase of a session step over the checkpoint-free median (same run);",
         "per-ckpt = that x K; wait = event-timed slot/state wait per session step; replay = host replay of the last session.",
         "",
         f"{'staging':8s} {'K':>3s} {'stall/step ms':>14s} {'% step':>7s} {'per-ckpt ms':>12s} {'wait ms':>8s} {'thr ratio':>10s} "
         f"{'D2H GB/s':>9s} {'session GB':>11s} {'replay ms':>10s} {'elem-upd G':>11s} {'kernel %HBM':>12s} {'SM MHz':>7s}"]
for d in rows:
    c, st = d["config"], d["stall"]
    lines.append(f"{c['staging']:8s} {c['K']:3d} {st['delta_ms_per_session_step_mean']:14.2f} {100 * st['delta_frac_of_step']:6.2f}% "
                 f"{st['delta_ms_per_session_step_mean'] * c['K']:12.1f} {st['wait_ms_per_session_step']:8.3f} "
                 f"{d['ckpt_free']['throughput_ratio']:10.4f} {d['d2h']['gbs']:9.1f} {d['d2h']['bytes_per_session'] / 1e9:11.1f} "
                 f"{d['replay']['host_ms_last_session']:10.0f} {d['replay']['element_updates_per_session'] / 1e9:11.2f} "
                 f"{100 * d['roofline']['frac']:11.1f}% {d['clocks']['sm_mhz']:7.0f}")
d = json.loads([l for l in open(P + f"{tag}_bench_llama7b_r8.json") if l.startswith("{")][-1])
st = d["stall"]
lines += ["", f"config 3 (Llama-2 7B, one rank of 8, n_r=842,301,952, K=8, 2x4096 tokens): stall "
              f"{st['delta_ms_per_session_step_mean']:.2f} ms/session step ({100 * st['delta_frac_of_step']:.2f}% of "
              f"{st['ckpt_free_step_ms_median']:.0f} ms), thr ratio {d['ckpt_free']['throughput_ratio']:.4f}, D2H "
              f"{d['d2h']['gbs']:.1f} GB/s, fused kernel {d['roofline']['achieved']:.0f} GB/s "
              f"({100 * d['roofline']['frac']:.1f}% HBM) @ {d['clocks']['sm_mhz']:.0f} MHz"]
s = [json.loads(l) for l in open(P + f"{tag}_schemes.jsonl") if l.startswith("{")]
lines += ["", "NEXT-3 scheme comparison (same harness, same box, one run; the paper's fig:stalltime analog): stall per checkpoint",
          "sync = blocking D2H snapshot of the full state; async-o = the snapshot overlaps the next F/B and its update waits;",
          "gockpt (paper, blocking) = parts from live memory, every update waits for its gradient slice (P:312-314);",
          "gockpt (ring) = this build's default (pre-update pack into an HBM ring); gockpt-O (direct) = GoCkpt-O (P:329-333).", ""]
for d in s:
    c, st = d["config"], d["stall"]
    name = c["scheme"] + ("" if c["scheme"] != "gockpt" else
                          {"direct": "-O (direct)", "ring": " (ring)", "blocking": " (paper, blocking)"}[c["staging"]])
    per = st["delta_ms_per_session_step_mean"] * (1 if c["scheme"] != "gockpt" else c["K"])
    same = st.get("delta_ms_vs_plain_steps_same_intervals")
    same_s = (f"   (vs plain steps of the same intervals: "
              f"{same * (1 if c['scheme'] != 'gockpt' else c['K']):8.2f} ms/ckpt)" if same is not None else "")
    lines.append(f"{c['workload'][:32]:32s} {name:26s} {per:9.2f} ms/ckpt   throughput ratio "
                 f"{d['ckpt_free']['throughput_ratio']:.4f}   step {st['ckpt_free_step_ms_median']:.1f} ms" + same_s)
open(P + f"{tag}_k_sweep_and_schemes.txt", "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
