#!/bin/bash
# Replay kernel with packed FFMA2/FMUL2/FADD2 arithmetic vs the scalar form; ncu; fast-math + parity tests.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
out=gpurun_out/r02_replay5.jsonl; : > $out
for impl in p r; do
  for nk in "124439808 8" "124439808 4" "124439808 16" "842301952 8" "842301952 4"; do
    set -- $nk
    r=$(GCK_REPLAY_IMPL=$impl GCK_N=$1 GCK_K=$2 timeout 300 python scripts/microbench_replay.py 2>&1 | tail -1)
    echo "{\"impl\": \"$impl\", \"r\": $r}" >> $out
  done
done
cat $out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:replay -s 2 -c 1 \
   -o gpurun_out/replay_v5 -f python scripts/microbench_replay.py > gpurun_out/ncu_replay_v5.log 2>&1; echo "ncu rc=$?"
timeout 1800 python -m pytest tests/test_gpu_fastmath.py -q -m gpu -x 2>&1 | tail -5 | tee gpurun_out/r02_fastmath_tests.txt
timeout 1800 python -m pytest tests/test_gpu_guard.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_faults.py -q -m gpu -x 2>&1 | tail -5 | tee gpurun_out/r02_replay5_tests.txt
