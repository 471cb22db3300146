#!/bin/bash
# When does K matter? GPT-2 124M shard at SHORT steps (4 x 1024 tokens, ~5 ms) where one part's
# transfer no longer fits in a step unless K is large: K = 1..32, ring and direct staging.
python -c "import __graft_entry__ as g; g.build()" || exit 1
OUT=gpurun_out/short_step.jsonl
: > $OUT
for st in ring direct; do
for K in 1 2 4 8 16 32; do
  timeout 600 python bench.py --tokens 4096 --K $K --interval $((2 * K + 8)) --steps 3 --warmup 3 --staging $st \
      --no-e2e --no-cpu-baseline >> $OUT 2>> gpurun_out/short_step.err || echo "K=$K $st failed" >&2
done; done
python - <<'PY'
import json
for l in open("gpurun_out/short_step.jsonl"):
    if not l.startswith("{"): continue
    d = json.loads(l); c = d["config"]; st = d["stall"]
    print(c["staging"], c["K"], "step %.2f ms" % st["ckpt_free_step_ms_median"], "stall/step %.2f ms (%.1f%%)" % (st["delta_ms_per_session_step_mean"], 100 * st["delta_frac_of_step"]),
          "wait %.3f" % st["wait_ms_per_session_step"], "thr %.4f" % d["ckpt_free"]["throughput_ratio"], "recK", d["model"]["recommended_K"])
PY
