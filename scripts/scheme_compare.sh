#!/bin/bash
# NEXT-3: the paper's stall comparison (fig:stalltime) on B200, same harness, same run.
python -c "import __graft_entry__ as g; g.build()" || exit 1
OUT=gpurun_out/schemes.jsonl
: > $OUT
run() { timeout 900 python bench.py "$@" --no-cpu-baseline --no-e2e >> $OUT 2>> gpurun_out/schemes.err || echo "failed: $*" >&2; }
for m in "--model gpt2-small --interval 50 --steps 3" "--model llama2-13b --shard-of 8 --interval 16 --steps 2"; do
  run $m --scheme sync
  run $m --scheme async-o
  run $m --scheme gockpt --staging ring
  run $m --scheme gockpt --staging direct
  run $m --scheme gockpt --staging blocking
done
python - <<'PY'
import json
rows=[json.loads(l) for l in open("gpurun_out/schemes.jsonl") if l.startswith("{")]
for d in rows:
    c=d["config"]; st=d["stall"]
    name = c["scheme"] + ("" if c["scheme"] != "gockpt" else {"direct": "-O (direct)", "ring": " (ring)", "blocking": " (paper, blocking)"}[c["staging"]])
    print(f'{c["workload"][:28]:28s} {name:20s} stall/ckpt {sum([st["delta_ms_per_session_step_mean"]]) * (1 if c["scheme"]!="gockpt" else c["K"]):9.2f} ms  '
          f'max step delta {st["delta_ms_per_session_step_max"]:8.2f} ms  thr ratio {d["ckpt_free"]["throughput_ratio"]:.4f}  step {st["ckpt_free_step_ms_median"]:.1f} ms')
PY
