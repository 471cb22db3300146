#!/bin/bash
# Replay-kernel variants: microbench (GPT-2 K=4/8/16, 7B rank-of-8 K=8) + replay parity tests.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
out=gpurun_out/r02_replay_variants.jsonl; : > $out
for cfg in s 0 1 2 3 4 5; do
  for nk in "124439808 8" "124439808 4" "124439808 16" "842301952 8"; do
    set -- $nk
    if [ $cfg = s ]; then impl=s; c=0; else impl=t; c=$cfg; fi
    r=$(GCK_REPLAY_IMPL=$impl GCK_REPLAY_CFG=$c GCK_N=$1 GCK_K=$2 timeout 300 python scripts/microbench_replay.py 2>&1 | tail -1)
    echo "{\"cfg\": \"$cfg\", \"r\": $r}" >> $out
  done
done
cat $out
timeout 1200 python -m pytest tests/test_gpu_guard.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -m gpu -x 2>&1 | tail -5 | tee gpurun_out/r02_replay_tests.txt
