#!/bin/bash
# Transfer-balanced partition plan: GPU parity over both plans, then bench lines equal vs balanced.
mkdir -p gpurun_out/plan
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 2400 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -3 | tee gpurun_out/plan/parity.txt
run() {  # name, args...
  local name=$1; shift
  timeout 1800 python bench.py "$@" --step-log gpurun_out/plan/$name.steps.jsonl > gpurun_out/plan/$name.json 2> gpurun_out/plan/$name.err
  echo "$name rc=$? $(tail -c 200 gpurun_out/plan/$name.json | head -c 200)"
}
run gpt2_balanced --plan balanced
for K in 4 6 8; do
  run c4_13b_r4_i50_k${K}_balanced --model llama2-13b --shard-of 4 --K $K --interval 50 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --plan balanced
done
run c4_13b_r4_i50_k6 --model llama2-13b --shard-of 4 --K 6 --interval 50 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline
