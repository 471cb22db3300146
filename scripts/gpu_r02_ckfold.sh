#!/bin/bash
# Drain verification folded into the fused kernel's pack warp: GPU tests that exercise it, then the
# 13B/4 and GPT-2 lines it is meant to improve.
mkdir -p gpurun_out/ckfold
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 2400 python -m pytest tests/test_gpu_faults.py tests/test_gpu_parity.py tests/test_gpu_guard.py tests/test_gpu_drain_cache.py tests/test_gpu_fullsize.py -q -m gpu -x 2>&1 | tail -3 | tee gpurun_out/ckfold/tests.txt
run() {  # name, args...
  local name=$1; shift
  timeout 1800 python bench.py "$@" --step-log gpurun_out/ckfold/$name.steps.jsonl > gpurun_out/ckfold/$name.json 2> gpurun_out/ckfold/$name.err
  echo "$name rc=$? $(tail -c 120 gpurun_out/ckfold/$name.json | head -c 120)"
}
run default
run c4_13b_r4_i50_k8 --model llama2-13b --shard-of 4 --K 8 --interval 50 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline
run c4_13b_r4_i50_k8_noverify --model llama2-13b --shard-of 4 --K 8 --interval 50 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --verify-drain 0
run c4_13b_r4_i50_k6_balanced --model llama2-13b --shard-of 4 --K 6 --interval 50 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --plan balanced
