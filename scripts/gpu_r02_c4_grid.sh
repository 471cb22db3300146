#!/bin/bash
# Completes SURVEY §8(d) C4's grid at 4 ranks: K = 3, 6, 12 at 2048 tokens and the 4 x 4096-token regime.
mkdir -p gpurun_out/grid
python -c "import __graft_entry__ as g; g.build()" || exit 1
run() {  # name, args...
  local name=$1; shift
  timeout 1800 python bench.py "$@" --step-log gpurun_out/grid/$name.steps.jsonl > gpurun_out/grid/$name.json 2> gpurun_out/grid/$name.err
  echo "$name rc=$?"
}
C="--model llama2-13b --shard-of 4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
for K in 3 6 12; do run c4_13b_r4_i50_k$K $C --K $K --interval 50; done
for K in 2 4 8 16; do run c4_13b_r4_t16k_k$K $C --K $K --tokens 16384 --interval 20; done
