#!/bin/bash
# Replay kernel: front/back interleaved unit order (GCK_REPLAY_MIX=1) vs the default order, same job.
mkdir -p gpurun_out/mix
python -c "import __graft_entry__ as g; g.build()" || exit 1
out=gpurun_out/mix/replay_mix.jsonl; : > $out
for rep in 1 2; do
for cfg in "0 64" "1 64" "1 16" "1 8"; do
  set -- $cfg
  for nk in "124439808 8" "124439808 4" "124439808 16" "842301952 8"; do
    set -- $cfg $nk
    echo "{\"mix\": $1, \"ctas\": $2, \"r\": $(GCK_REPLAY_MIX=$1 GCK_REPLAY_CTAS_PER_SM=$2 GCK_N=$3 GCK_K=$4 timeout 300 python scripts/microbench_replay.py 2>&1 | tail -1)}" >> $out
  done
done
done
cat $out
GCK_REPLAY_MIX=1 timeout 1200 python -m pytest tests/test_gpu_guard.py tests/test_gpu_fullsize.py -q -m gpu -x 2>&1 | tail -2 | tee gpurun_out/mix/tests_mix.txt
