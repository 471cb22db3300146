#!/bin/bash
# C4 at 8 ranks (13B rank-of-8, n_r = 1.63G) on the final tree: the SURVEY's K grid at 2048 tokens, interval 50.
mkdir -p gpurun_out/r8
python -c "import __graft_entry__ as g; g.build()" || exit 1
for K in 2 3 4 6 8 12 16; do
  timeout 1200 python bench.py --model llama2-13b --shard-of 8 --K $K --interval 50 --steps 3 --warmup 3 --no-e2e \
      --no-cpu-baseline --step-log gpurun_out/r8/c4_13b_r8_i50_k$K.steps.jsonl > gpurun_out/r8/c4_13b_r8_i50_k$K.json \
      2> gpurun_out/r8/c4_13b_r8_i50_k$K.err
  echo "k$K rc=$?"
done
