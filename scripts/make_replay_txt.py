"""profiles/r02_replay_kernel.txt from the replay microbench JSONL files in gpurun_out/ (CPU)."""
import json
import os

HEAD = open(os.path.join(os.path.dirname(__file__), "replay_txt_head.txt")).read()
LEGEND = {
    "r02_replay4.jsonl": "t = 3-way unrolled + cp.async state prefetch, u = 3-way unrolled, r = kept kernel "
                         "(minb = CTAs/SM register bound of t/u)",
    "r02_replay7.jsonl": "b = TMA-pipelined + packed arithmetic (T0 4096x16 warps, T1 2048x16, T2 4096x8, "
                         "T3 2048x8), p = kept kernel with packed arithmetic, r = kept kernel",
    "r02_replay8.jsonl": "f4/f5/f6 = 4 elements per thread at 4/5/6 CTAs per SM, p = packed, r = kept kernel",
    "r02_replay9.jsonl": "pref = 0 kept kernel, 1 + L2 bulk prefetch of the warp's next group, 2 + the "
                         "gradient two steps ahead (each twice)",
    "r02_replay10.jsonl": "coalesced = 0 the 8-consecutive-element kernel, 1 the warp-coalesced default "
                          "(each twice)",
    "r02_replay11_grid_a.jsonl": "ctas_per_sm = grid size of the coalesced kernel (grid-stride), twice",
    "r02_replay11.jsonl": "ctas_per_sm, larger grids (100000 = one group per thread)",
    "r02_replay12.jsonl": "FINAL: t = the kernel as committed (coalesced, 64 CTAs/SM), s = the round-1 kernel with "
                          "the same grid; twice",
    "r02_replay_final.jsonl": "t = the kept kernel as committed (default), s = the round-1 kernel "
                              "(replay_generic_kernel, GCK_REPLAY_IMPL=s), alternated twice",
}
lines = [HEAD.rstrip(), "", "Microbench (us mean / GB/s / frac of 6555.2); each file is one gpurun job:"]
for f, leg in LEGEND.items():
    p = os.path.join("gpurun_out", f)
    if not os.path.exists(p):
        continue
    lines.append(f"  {f}: {leg}")
    for l in open(p):
        try:
            d = json.loads(l)
        except ValueError:
            continue
        r = d["r"]
        tag = str(d.get("impl", d.get("pref", d.get("coalesced", d.get("ctas_per_sm", ""))))) + (f" minb{d['minb']}" if "minb" in d else "") + (f" T{d['T']}" if "T" in d else "")
        lines.append(f"    {tag:9s} n={r['n']:>11,d} K={r['K']:>2d}  {r['us_mean']:8.1f} us  {r['gbs']:7.1f} GB/s  "
                     f"{r['gbs'] / 6555.2:.3f}")
open("profiles/r02_replay_kernel.txt", "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
