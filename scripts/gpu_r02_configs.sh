#!/bin/bash
# BASELINE configs as bench lines (round 2): C1 flat-1M (1 ms spin and 0 ms), C3 Llama-2 7B rank-of-8 at
# interval 100 (3 timed sessions), C4 Llama-2 13B at 2 ranks (n_r = 6.5e9 > 2^32; R=1 ring K=2/3, direct
# K=2/3, streaming replay K=16 B=4) and at 4 ranks (K sweep), each with its per-step JSONL log.
mkdir -p gpurun_out/cfg
python -c "import __graft_entry__ as g; g.build()" || exit 1
run() {  # name, args...
  local name=$1; shift
  timeout 1500 python bench.py "$@" --step-log gpurun_out/cfg/$name.steps.jsonl > gpurun_out/cfg/$name.json 2> gpurun_out/cfg/$name.err
  echo "$name rc=$? $(tail -c 300 gpurun_out/cfg/$name.json | head -c 300)"
}
run c1_spin1 --model flat-1m --K 4 --interval 20 --steps 5 --warmup 3 --spin-ms 1
run c1_spin0 --model flat-1m --K 4 --interval 20 --steps 5 --warmup 3 --spin-ms 0
run c3_7b_r8_i100 --model llama2-7b --shard-of 8 --K 8 --interval 100 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline
run c4_13b_r2_k2_ring1 --model llama2-13b --shard-of 2 --K 2 --ring-slots 1 --interval 20 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline
run c4_13b_r2_k3_ring1 --model llama2-13b --shard-of 2 --K 3 --ring-slots 1 --interval 20 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline
run c4_13b_r2_k2_direct --model llama2-13b --shard-of 2 --K 2 --staging direct --interval 20 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline
run c4_13b_r2_k3_direct --model llama2-13b --shard-of 2 --K 3 --staging direct --interval 20 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline
run c4_13b_r2_k16_stream4 --model llama2-13b --shard-of 2 --K 16 --replay-mode stream --stream-buffers 4 --interval 20 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline
for K in 2 4 8 16; do
  run c4_13b_r4_k$K --model llama2-13b --shard-of 4 --K $K --interval 20 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline
done
free -g | head -2
