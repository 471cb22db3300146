#!/bin/bash
# Replay kernel: streaming cache hints (.cs loads + stores / .cs stores only) vs none, same job, twice.
mkdir -p gpurun_out/cs
python -c "import __graft_entry__ as g; g.build()" || exit 1
out=gpurun_out/cs/replay_cs.jsonl; : > $out
for rep in 1 2; do
for cs in 0 1 2; do
  for nk in "124439808 8" "124439808 4" "124439808 16" "842301952 8"; do
    set -- $nk
    echo "{\"cs\": $cs, \"r\": $(GCK_REPLAY_CS=$cs GCK_N=$1 GCK_K=$2 timeout 300 python scripts/microbench_replay.py 2>&1 | tail -1)}" >> $out
  done
done
done
cat $out
