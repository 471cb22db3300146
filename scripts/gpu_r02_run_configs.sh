#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_fastmath.py tests/test_gpu_guard.py -q -m gpu 2>&1 | tail -3 | tee gpurun_out/r02_final_kernel_tests.txt
for impl in t s t s; do
  for nk in "124439808 8" "124439808 4" "842301952 8"; do
    set -- $nk
    echo "{\"impl\": \"$impl\", \"r\": $(GCK_REPLAY_IMPL=$impl GCK_N=$1 GCK_K=$2 timeout 300 python scripts/microbench_replay.py 2>&1 | tail -1)}"
  done
done > gpurun_out/r02_replay_final.jsonl
timeout 600 ncu --set full --import-source on --clock-control none -k regex:replay -s 2 -c 1 \
   -o gpurun_out/replay_final -f python scripts/microbench_replay.py > gpurun_out/ncu_replay_final.log 2>&1
bash scripts/gpu_r02_configs.sh
