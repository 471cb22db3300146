#!/bin/bash
# Replay kernel: 64- and 128-thread CTAs around the 256 default (grid scaled to the same threads), twice.
mkdir -p gpurun_out/blk
python -c "import __graft_entry__ as g; g.build()" || exit 1
out=gpurun_out/blk/replay_blk2.jsonl; : > $out
for rep in 1 2; do
for cfg in "256 64" "128 64" "128 32" "128 128" "64 64" "64 32"; do
  set -- $cfg
  for nk in "124439808 8" "124439808 4" "842301952 8"; do
    set -- $cfg $nk
    echo "{\"blk\": $1, \"ctas\": $2, \"r\": $(GCK_REPLAY_BLOCK=$1 GCK_REPLAY_CTAS_PER_SM=$2 GCK_N=$3 GCK_K=$4 timeout 300 python scripts/microbench_replay.py 2>&1 | tail -1)}" >> $out
  done
done
done
