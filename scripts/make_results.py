"""Regenerate BASELINE.md's "## Results" section from the raw lines in profiles/ (round tag argv[1])."""
import json
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
P = "profiles/"
try:
    HBM = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"]
except (OSError, KeyError, ValueError):
    HBM = 6500.6


def last_json(path):
    return json.loads([l for l in open(path) if l.startswith("{")][-1])


d = last_json(P + f"{tag}_bench_default.json")
ref = last_json(P + f"{tag}_bench_reference.json")
q = [json.loads(l) for l in open(P + f"{tag}_k_sweep_llama13b_r8.jsonl") if l.startswith("{")]
l7 = last_json(P + f"{tag}_bench_llama7b_r8.json")
mf = last_json(P + f"{tag}_microbench_fused.json")
mr = last_json(P + f"{tag}_microbench_replay.json")
hr = last_json(P + f"{tag}_host_replay.json")
try:
    lg = last_json(P + f"{tag}_bench_long_20intervals.json")
    long_line = (f"- **Long run** (`{tag}_bench_long_20intervals.json`, 20 intervals = 1000 training steps, 20 sessions):\n"
                 f"  throughput ratio {lg['ckpt_free']['throughput_ratio']:.5f}, stall {lg['stall']['delta_ms_per_session_step_mean']:.2f} ms "
                 f"per session step ({100 * lg['stall']['delta_frac_of_step']:.2f}%), amortized "
                 f"{100 * lg['stall']['amortized_frac']:.3f}% of training time; fused kernel {100 * lg['roofline']['frac']:.1f}% HBM live.\n")
except (OSError, IndexError):
    long_line = ""


def row(name, gpus, K, x):
    st, r = x["stall"], x["roofline"]
    sess = r["session_launches"]["achieved_gbs"]
    if sess and x["config"].get("staging", "ring") != "ring":
        # lines measured before bench.py stopped counting slot bytes the direct-staging kernel never
        # writes: rescale to the kernel's own bytes (28n per launch)
        alg = r["session_launches"]["alg_bytes_per_launch_mean"]
        if alg > r["alg_bytes_per_launch"]:
            sess = sess * r["alg_bytes_per_launch"] / alg
    return (f"| {name} | {gpus} | {K} | {x['config'].get('staging', 'ring')} | {st['wait_ms_per_session_step']:.3f} / "
            f"{st['delta_ms_per_session_step_mean']:.2f} ms ({100 * st['delta_frac_of_step']:.2f}% of a "
            f"{st['ckpt_free_step_ms_median']:.1f} ms step) | {x['ckpt_free']['throughput_ratio']:.4f} | "
            f"{x['d2h']['gbs']:.1f} ({100 * x['d2h']['frac']:.1f}%) | {100 * r['frac']:.1f}% plain"
            + (f", {100 * sess / r['peak']:.1f}% session" if sess else "") + f" @ {x['clocks']['sm_mhz']:.0f} MHz | "
            f"{x['replay']['host_ms_last_session']:.0f} ms |")


SCH = [json.loads(l) for l in open(P + f"{tag}_schemes.jsonl") if l.startswith("{")]


def _per_ckpt(d):
    st, c = d["stall"], d["config"]
    return st["delta_ms_per_session_step_mean"] * (1 if c["scheme"] != "gockpt" else c["K"])


def _name(c):
    return {"sync": "Sync", "async-o": "Async-O"}.get(c["scheme"]) or {
        "ring": "ring GoCkpt", "direct": "GoCkpt-O", "blocking": "paper-faithful GoCkpt (blocking gradient D2H)"}[c["staging"]]


def schemes(prefix):
    return ", ".join(f"{_name(d['config'])} {_per_ckpt(d):.1f} ms" for d in SCH if d["config"]["workload"].startswith(prefix))


_l13 = {_name(d["config"]): _per_ckpt(d) for d in SCH if d["config"]["workload"].startswith("Llama-2 13B")}
ratio_o = _l13["GoCkpt-O"] / _l13["Async-O"]

out = f"""## Results (round 1, measured on one B200 via gpurun; raw lines in `profiles/{tag}_*`)

Stall = event-timed slot/state wait per session step / mean step-time increase of a session
step over the checkpoint-free median of the same run. Throughput ratio = tokens/s with GoCkpt ÷
checkpoint-free tokens/s, same run (both ±0.5% run noise). HBM % = fused-kernel algorithmic
bytes ÷ live CUDA-event time ÷ the measured HBM copy peak in MEASURED_PEAKS.json ({HBM} GB/s this round;
bench.py reads it at run time). Link % against the best-of-5 1 GiB
D2H of the same run. Parity: every config below is also a `-m gpu` test — checkpoint bit-identical
to the GPU's own synchronous snapshot over all elements and to the oracle on sampled windows.

| Config | GPUs | K | staging | Stall wait / Δ per session step | Thr. vs ckpt-free | D2H GB/s (% link) | Fused kernel HBM | Host replay |
|---|---|---|---|---|---|---|---|---|
{row("C2 GPT-2 124M (bench.py default), interval 50, 16×1024 tok", 1, 8, d)}
{row("C3 Llama-2 7B, one rank of 8 (n_r=842M), 2×4096 tok", "1 (rank of 8)", 8, l7)}
""" + "\n".join(row("C4 Llama-2 13B, one rank of 8 (n_r=1.63G), 2048 tok", "1 (rank of 8)", x["config"]["K"], x)
                for x in q) + f"""

(C3/C4 rows: the final kernel at the power-capped ~1.35–1.40 GHz these GEMM-heavy steps run at.)

- **Headline (bench.py default, C2):** {d['value']:.0f} tokens/s with a consistent checkpoint every 50
  steps vs {d['ckpt_free']['value']:.0f} checkpoint-free (ratio {d['ckpt_free']['throughput_ratio']:.4f}) at
  {d['clocks']['sm_mhz']:.0f} MHz (power-capped); e2e (gradient H2D from pinned host + result read each step)
  {d['e2e']['value']:.0f} tokens/s; {d['gpu_launches']} of our kernels in the timed region.
{long_line}- **Fused AdamW+pack kernel:** {mf['plain_us_mean']:.0f} µs = {mf['plain_gbs']:.0f} GB/s =
  {100 * mf['plain_gbs'] / HBM:.1f}% of the measured HBM copy in isolation (session launches
  {mf['session_gbs']:.0f} GB/s); live in the bench {100 * d['roofline']['frac']:.1f}%; ncu: DRAM bytes = the algorithmic 28n;
  a plain 8-stream copy of the same pattern tops out at 5.6–6.16 TB/s (`{tag}_stream8.txt`).
- **Replay:** host pool {hr['runs'][-1]['ms']:.1f} ms for {hr['element_updates'] / 1e6:.0f}M element-updates at
  {hr['runs'][-1]['threads']} threads = {hr['runs'][-1]['gbs']:.0f} GB/s = {100 * hr['runs'][-1]['frac_of_triad']:.0f}% of the box's STREAM
  triad ({hr['runs'][-1]['triad_gbs']:.0f} GB/s); 1 thread {hr['runs'][0]['ms']:.0f} ms. GPU replay kernel {mr['us_mean']:.0f} µs =
  {mr['gbs']:.0f} GB/s ({100 * mr['gbs'] / HBM:.0f}% of HBM) — but the bound is issue, not HBM: 45.6 warp-instructions
  per 32 element-updates, ncu issue-active 80%, 79% of the issue roofline (553 µs at 1.9 GHz); a part-interleaved
  variant was slower (`{tag}_replay_interleave_experiment.txt`).
- **CPU oracle on one host core** (`--impl reference`, 2^20-element sample scaled): {ref['value']:.0f}
  tokens/s-equivalent; {d['cpu_baseline']['value']:.0f} with the 2^24 sample of the bench's cpu_baseline leg
  (AdamW + capture + replay only, no F/B).
- **Stall vs the paper's schemes on B200** (NEXT-3, `{tag}_k_sweep_and_schemes.txt`, one run), per
  checkpoint (session-step delta × K vs the checkpoint-free run): GPT-2 — {schemes('GPT-2')};
  Llama-2 13B rank-of-8 shard — {schemes('Llama-2 13B')}. GoCkpt-O's stall is {100 * ratio_o:.0f}% of
  Async-O's on the 13B shard (the paper reports 0.5–10% on V100S, P:452).
- **C5 D2H sweep** (`{tag}_d2h_sweep.txt`): copy engine 56–57 GB/s from 16 MiB to 8 GiB;
  zero-copy 50–52.7 GB/s, 20–44 GB/s under a concurrent GEMM; 4 MiB chunks (P:362) cost ~5%.
- **Persistence** (NEXT-1, `{tag}_persist.txt`): 1.95 GB/s write, ~3 GB/s cold restore on the box's
  virtio disk (GPT-2 shard 0.77 s / 0.54 s; 7B rank shard 5.2 s / 3.2 s).
- **Replay modes** (`{tag}_replay_modes.txt`, `{tag}_persist_modes.txt`): streaming host replay
  (B = 2 recycled slice buffers: pinned arena 16n instead of 19n) ratio 0.9967 vs 0.9959 batch, D2H
  56.0 vs 56.8 GB/s on GPT-2/K=8; at 13B rank-of-8/K=16 B=2 starves the GPU queue (5–8 ms stall per
  session step) while the default B=4 (arena 20n instead of 27n) stalls 1.0 ms, on par with the batch
  replay (`{tag}_stream_13b_k16.txt`); replay-on-restore: finalize 3 ms instead of 31 ms, file 2.36 vs 1.49 GB,
  persist 1.19 vs 0.76 s, cold restore (GPU replay in place) 1.46 vs 0.54 s; restored bytes
  identical (CRC) in every mode.
- **Sanitizers** (`{tag}_sanitizers.txt`, `{tag}_host_sanitizers.txt`, `{tag}_gpu_tsan.txt`): compute-sanitizer
  memcheck / racecheck / synccheck clean; ASan+UBSan and TSan clean on the host code and on the GPU
  session paths (eager / streaming / deferred replay, persist, abort).
- Multi-GPU (2/4/8) was not measured this round: gpurun provides one GPU. `bench.py` runs under
  torchrun (ZeRO-1 shards; NCCL RS/AG in the harness only); the host logic is covered by
  world-size-2 gloo tests.
"""
s = open("BASELINE.md").read()
s = s[:s.index("## Results")] + out
open("BASELINE.md", "w").write(s)
print(out[:1500])
