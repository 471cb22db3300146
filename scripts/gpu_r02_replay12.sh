#!/bin/bash
# The replay kernel as committed (warp-coalesced, 64 CTAs/SM) vs the round-1 kernel, same job; ncu; tests.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
out=gpurun_out/r02_replay12.jsonl; : > $out
for rep in 1 2; do
for impl in t s; do
  for nk in "124439808 8" "124439808 4" "124439808 16" "842301952 8" "842301952 4"; do
    set -- $nk
    echo "{\"impl\": \"$impl\", \"r\": $(GCK_REPLAY_IMPL=$impl GCK_N=$1 GCK_K=$2 timeout 300 python scripts/microbench_replay.py 2>&1 | tail -1)}" >> $out
  done
done
done
cat $out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:replay -s 2 -c 1 \
   -o gpurun_out/replay_final2 -f python scripts/microbench_replay.py > gpurun_out/ncu_replay_final2.log 2>&1; echo "ncu rc=$?"
timeout 1500 python -m pytest tests/test_gpu_guard.py tests/test_gpu_fullsize.py tests/test_gpu_parity.py tests/test_gpu_huge.py -q -m gpu 2>&1 | tail -3 | tee gpurun_out/r02_replay12_tests.txt
