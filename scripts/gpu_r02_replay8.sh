#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
out=gpurun_out/r02_replay8.jsonl; : > $out
for impl in r s; do
  for nk in "124439808 8" "124439808 4" "842301952 8"; do
    set -- $nk
    r=$(GCK_REPLAY_IMPL=$impl GCK_N=$1 GCK_K=$2 timeout 300 python scripts/microbench_replay.py 2>&1 | tail -1)
    echo "{\"impl\": \"$impl\", \"r\": $r}" >> $out
  done
done
cat $out
