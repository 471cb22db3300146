#!/bin/bash
# Final-tree refresh of the BASELINE config lines that do not need the 13B/2 shard (C1, C3, C4 at 4
# ranks incl. streaming replay at K = 8 / 16), plus the drain-cache GPU test.
mkdir -p gpurun_out/cfgf
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests/test_gpu_drain_cache.py -q -m gpu 2>&1 | tail -3 | tee gpurun_out/cfgf/drain_cache_test.txt
run() {  # name, args...
  local name=$1; shift
  timeout 1800 python bench.py "$@" --step-log gpurun_out/cfgf/$name.steps.jsonl > gpurun_out/cfgf/$name.json 2> gpurun_out/cfgf/$name.err
  echo "$name rc=$? $(tail -c 200 gpurun_out/cfgf/$name.json | head -c 200)"
}
run c1_spin1 --model flat-1m --K 4 --interval 20 --steps 5 --warmup 3 --spin-ms 1
run c1_spin0 --model flat-1m --K 4 --interval 20 --steps 5 --warmup 3 --spin-ms 0
run c3_7b_r8_i100 --model llama2-7b --shard-of 8 --K 8 --interval 100 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline
for K in 2 4 8 16; do
  run c4_13b_r4_k$K --model llama2-13b --shard-of 4 --K $K --interval 20 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline
done
for K in 8 16; do
  run c4_13b_r4_k${K}_stream4 --model llama2-13b --shard-of 4 --K $K --replay-mode stream --stream-buffers 4 --interval 20 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline
done
