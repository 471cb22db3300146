#!/bin/bash
# Packed arithmetic in every replay variant: v2 (p), scalar v2 (r), cp.async ring D=2/3/4 (c), unrolled (t/u).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
out=gpurun_out/r02_replay6.jsonl; : > $out
for cfg in "p 3" "r 3" "c 2" "c 3" "c 4" "t 3" "u 3"; do
  set -- $cfg; impl=$1; D=$2
  for nk in "124439808 8" "124439808 4" "842301952 8"; do
    set -- $nk
    r=$(GCK_REPLAY_IMPL=$impl GCK_REPLAY_D=$D GCK_REPLAY_MINB=3 GCK_N=$1 GCK_K=$2 timeout 300 python scripts/microbench_replay.py 2>&1 | tail -1)
    echo "{\"impl\": \"$impl\", \"D\": $D, \"r\": $r}" >> $out
  done
done
cat $out
GCK_REPLAY_IMPL=c GCK_REPLAY_D=3 timeout 600 ncu --set full --import-source on --clock-control none -k regex:replay -s 2 -c 1 \
   -o gpurun_out/replay_v6c -f python scripts/microbench_replay.py > gpurun_out/ncu_replay_v6c.log 2>&1; echo "ncu rc=$?"
