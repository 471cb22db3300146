#!/bin/bash
# BASELINE config 4 (K sweep 2..16: stall vs consistency-replay cost) on one B200 emulating one
# rank of an 8-GPU Llama-2 13B ZeRO-1 job (n_r = 1,626,983,424), short step (1 x 2048 tokens),
# ring and direct staging. Also config 3 (Llama-2 7B rank shard, K=8). JSON lines in gpurun_out/.
python -c "import __graft_entry__ as g; g.build()" || exit 1
OUT=gpurun_out/k_sweep.jsonl
: > $OUT
for st in ${STAGINGS:-ring direct}; do
for K in ${KS:-2 3 4 6 8 12 16}; do
  timeout 900 python bench.py --model llama2-13b --shard-of 8 --K $K --interval $((K + 8)) --steps 2 --warmup 3 \
      --staging $st --no-e2e --no-cpu-baseline >> $OUT 2> gpurun_out/k_sweep_K$K.err || echo "K=$K $st failed" >&2
done; done
timeout 900 python bench.py --model llama2-7b --shard-of 8 --K 8 --interval 20 --steps 2 --warmup 3 \
    --no-e2e --no-cpu-baseline > gpurun_out/llama7b_r8.json 2> gpurun_out/llama7b_r8.err
