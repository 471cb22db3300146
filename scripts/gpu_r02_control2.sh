#!/bin/bash
mkdir -p gpurun_out/ctl gpurun_out/cfg
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_dist_smoke.py -q -m gpu -k nccl 2>&1 | tail -60 > gpurun_out/ctl/nccl_test.txt
bash scripts/gpu_r02_replay9.sh
for K in 8 16; do
  timeout 1500 python bench.py --model llama2-13b --shard-of 4 --K $K --interval 20 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline \
     --step-log gpurun_out/cfg/c4_13b_r4_k${K}_fold.steps.jsonl > gpurun_out/cfg/c4_13b_r4_k${K}_fold.json 2> gpurun_out/cfg/c4_13b_r4_k${K}_fold.err
  tail -c 200 gpurun_out/cfg/c4_13b_r4_k${K}_fold.json
done
