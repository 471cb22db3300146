#!/bin/bash
# Where the ~2% per-session-step floor at 13B/4 comes from: the same lines with the drain verification off.
mkdir -p gpurun_out/floor
python -c "import __graft_entry__ as g; g.build()" || exit 1
run() {  # name, args...
  local name=$1; shift
  timeout 1800 python bench.py "$@" --step-log gpurun_out/floor/$name.steps.jsonl > gpurun_out/floor/$name.json 2> gpurun_out/floor/$name.err
  echo "$name rc=$? $(tail -c 120 gpurun_out/floor/$name.json | head -c 120)"
}
run c4_13b_r4_i50_k8_noverify --model llama2-13b --shard-of 4 --K 8 --interval 50 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --verify-drain 0
run c4_13b_r4_i50_k4_balanced_noverify --model llama2-13b --shard-of 4 --K 4 --interval 50 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --verify-drain 0 --plan balanced
run c4_13b_r4_i50_k16_balanced --model llama2-13b --shard-of 4 --K 16 --interval 50 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --plan balanced
