#!/bin/bash
# NEXT-4 automatic K (--K 0: the library picks K from the measured step time and link) under both plans, 13B/4.
mkdir -p gpurun_out/autok
python -c "import __graft_entry__ as g; g.build()" || exit 1
for plan in equal balanced; do
  timeout 1800 python bench.py --model llama2-13b --shard-of 4 --K 0 --interval 50 --steps 3 --warmup 3 --no-e2e \
      --no-cpu-baseline --plan $plan --step-log gpurun_out/autok/c4_13b_r4_i50_kauto_$plan.steps.jsonl \
      > gpurun_out/autok/c4_13b_r4_i50_kauto_$plan.json 2> gpurun_out/autok/c4_13b_r4_i50_kauto_$plan.err
  echo "$plan rc=$?"
done
