#!/bin/bash
# tests + ncu of the fused kernel + bench, one gpurun call
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -5
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_adamw_pack -s 2 -c 3 \
    -o gpurun_out/fused -f python scripts/profile_fused.py > gpurun_out/ncu_full.log 2>&1
for impl in ${IMPLS:-tma simple}; do
  GCK_FUSED_IMPL=$impl timeout 600 python bench.py ${BENCH_ARGS} > gpurun_out/bench_$impl.json 2> gpurun_out/bench_$impl.err
  echo "== $impl"; python - <<PY
import json
d=json.loads(open("gpurun_out/bench_$impl.json").read().strip().splitlines()[-1])
print({k:d[k] for k in ("value","ms_per_step")}, d["roofline"]["achieved"], d["roofline"]["frac"], d["roofline"]["mean_launch_us"], d["stall"], d["d2h"]["gbs"], d["replay"], d["ckpt_free"], d["e2e"] and d["e2e"]["value"])
PY
done
