"""Summarise an ncu --set full report of fused_adamw_pack and a launch-list CSV into profiles/.

python scripts/summarize_ncu.py <fused.ncu-rep> <launches.csv> <round tag> <n>
Writes profiles/<tag>_fused_adamw_pack_ncu.txt, profiles/<tag>_launches.txt and
profiles/fused_adamw_pack_ncu.json (read by bench.py for roofline.traffic).
"""
import collections
import csv
import io
import json
import subprocess
import sys

rep, launches, tag, n = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4])
out_launches = sys.argv[5] if len(sys.argv) > 5 else f"profiles/{tag}_launches.txt"
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
           "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
           "lts__t_bytes.sum", "l1tex__t_bytes.sum"]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout if rep != "-" else ""
rows = list(csv.reader(io.StringIO(raw))) or [[], []]
hdr, units = rows[0], rows[1]
out, recs = [], []
for r in rows[2:]:
    rec = {"kernel": r[hdr.index("Kernel Name")]}
    for m in METRICS:
        if m in hdr:
            rec[m] = (r[hdr.index(m)], units[hdr.index(m)])
    recs.append(rec)
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1e-6, "ms": 1e-3, "ns": 1e-9, "s": 1}
lines = [f"ncu --set full --clock-control none, fused_adamw_pack at n={n} (bench config)", ""]
js = {"n": n, "launches": []}
for rec in recs:
    t = float(rec["gpu__time_duration.sum"][0].replace(",", "")) * scale[rec["gpu__time_duration.sum"][1]]
    rd = float(rec["dram__bytes_read.sum"][0].replace(",", "")) * scale[rec["dram__bytes_read.sum"][1]]
    wr = float(rec["dram__bytes_write.sum"][0].replace(",", "")) * scale[rec["dram__bytes_write.sum"][1]]
    pack = "<1>" in rec["kernel"] or "true" in rec["kernel"] or "kernel<1," in rec["kernel"]
    alg = 28 * n
    lines.append(f"{'pack ' if pack else 'plain'} {rec['kernel'][:70]}")
    lines.append(f"   time {t * 1e6:.1f} us  dram read {rd / 1e9:.4f} GB  write {wr / 1e9:.4f} GB  "
                 f"-> {(rd + wr) / t / 1e9:.0f} GB/s ; plain algorithmic bytes 28n = {alg / 1e9:.4f} GB")
    for m in METRICS[3:]:
        if m in rec:
            lines.append(f"   {m:60s} {rec[m][0]} {rec[m][1]}")
    js["launches"].append({"pack": pack, "time_s": t, "dram_read": rd, "dram_write": wr})
plain = [x for x in js["launches"] if not x["pack"]]
if plain:
    js["dram_bytes_per_launch"] = plain[0]["dram_read"] + plain[0]["dram_write"]
    js["note"] = "traffic of the plain (no-pack) launch, the dominant launch kind of a checkpoint interval"
if rep != "-":
    open(f"profiles/{tag}_fused_adamw_pack_ncu.txt", "w").write("\n".join(lines) + "\n")
    json.dump(js, open("profiles/fused_adamw_pack_ncu.json", "w"), indent=1)

print("\n".join(lines[:12]))
if launches == "-":
    sys.exit(0)
rows = list(csv.reader(open(launches)))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, mi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
tot, cnt = collections.defaultdict(float), collections.Counter()
for r in rows[hi + 1:]:
    if len(r) <= mi:
        continue
    v = float(r[mi].replace(",", "")) * {"ns": 1e-3, "us": 1, "ms": 1e3, "s": 1e6}[r[ui]]
    tot[r[ki][:90]] += v
    cnt[r[ki][:90]] += 1
T = sum(tot.values())
L = [f"ncu --metrics gpu__time_duration.sum --clock-control none (serialised, cold cache): {sum(cnt.values())} "
     f"launches, {T / 1e3:.1f} ms total", ""]
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    L.append(f"{v / 1e3:10.2f} ms {100 * v / T:6.2f}%  n={cnt[k]:6d}  mean {v / cnt[k]:9.1f} us  {k}")
gck = sum(v for k, v in tot.items() if "gck::" in k)
L.insert(1, f"share of our kernels (gck::*): {100 * gck / T:.2f}% of GPU time")
open(out_launches, "w").write("\n".join(L) + "\n")
print("\n".join(L[:6]))
