#!/bin/bash
# Replay kernel v3 (per-thread cp.async prefetch ring): D sweep vs register-prefetch v2 vs generic; ncu; tests.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
out=gpurun_out/r02_replay3.jsonl; : > $out
for cfg in "t 3" "t 2" "t 4" "r 3" "s 3"; do
  set -- $cfg; impl=$1; D=$2
  for nk in "124439808 8" "124439808 4" "124439808 16" "842301952 8"; do
    set -- $nk
    r=$(GCK_REPLAY_IMPL=$impl GCK_REPLAY_D=$D GCK_N=$1 GCK_K=$2 timeout 300 python scripts/microbench_replay.py 2>&1 | tail -1)
    echo "{\"impl\": \"$impl\", \"D\": $D, \"r\": $r}" >> $out
  done
done
cat $out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:replay -s 2 -c 1 \
   -o gpurun_out/replay_v3 -f python scripts/microbench_replay.py > gpurun_out/ncu_replay_v3.log 2>&1; echo "ncu rc=$?"
timeout 1800 python -m pytest tests/test_gpu_guard.py tests/test_gpu_faults.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -m gpu -x 2>&1 | tail -15 | tee gpurun_out/r02_replay3_tests.txt
