#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
out=gpurun_out/r02_replay11.jsonl; : > $out
for rep in 1; do
for c in 16 24 32 64 128 100000; do
  for nk in "124439808 8" "124439808 4" "842301952 8"; do
    set -- $nk
    echo "{\"ctas_per_sm\": $c, \"r\": $(GCK_REPLAY_CTAS_PER_SM=$c GCK_N=$1 GCK_K=$2 timeout 300 python scripts/microbench_replay.py 2>&1 | tail -1)}" >> $out
  done
done
done
cat $out
