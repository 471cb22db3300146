#!/bin/bash
# ncu --set full of the replay kernels (old grid-stride vs TMA variants) + the new fault / guard tests.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python -m pytest tests/test_gpu_faults.py tests/test_gpu_guard.py tests/test_gpu_fastmath.py -q -m gpu -x 2>&1 | tail -15 | tee gpurun_out/r02_fault_guard_tests.txt
for cfg in s 0 4; do
  if [ $cfg = s ]; then impl=s; c=0; else impl=t; c=$cfg; fi
  GCK_REPLAY_IMPL=$impl GCK_REPLAY_CFG=$c timeout 600 ncu --set full --import-source on --clock-control none -k regex:replay -s 2 -c 1 \
     -o gpurun_out/replay_$cfg -f python scripts/microbench_replay.py > gpurun_out/ncu_replay_$cfg.log 2>&1
  echo "ncu $cfg rc=$?"
done
