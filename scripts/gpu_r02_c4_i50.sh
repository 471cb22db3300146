#!/bin/bash
# BASELINE config 4 at 4 ranks with the paper's checkpoint interval (50 steps): K = 2, 4, 8, 16.
mkdir -p gpurun_out/cfgf
python -c "import __graft_entry__ as g; g.build()" || exit 1
run() {  # name, args...
  local name=$1; shift
  timeout 1800 python bench.py "$@" --step-log gpurun_out/cfgf/$name.steps.jsonl > gpurun_out/cfgf/$name.json 2> gpurun_out/cfgf/$name.err
  echo "$name rc=$? $(tail -c 200 gpurun_out/cfgf/$name.json | head -c 200)"
}
for K in 2 4 8 16; do
  run c4_13b_r4_i50_k$K --model llama2-13b --shard-of 4 --K $K --interval 50 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline
done
