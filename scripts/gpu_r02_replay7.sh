#!/bin/bash
# TMA-pipelined replay with packed arithmetic: 4 configurations vs v2 packed / scalar; ncu of the best TMA.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
out=gpurun_out/r02_replay7.jsonl; : > $out
for cfg in "b 0" "b 1" "b 2" "b 3" "p 0" "r 0"; do
  set -- $cfg; impl=$1; T=$2
  for nk in "124439808 8" "124439808 4" "124439808 16" "842301952 8"; do
    set -- $nk
    r=$(GCK_REPLAY_IMPL=$impl GCK_REPLAY_TMA=$T GCK_N=$1 GCK_K=$2 timeout 300 python scripts/microbench_replay.py 2>&1 | tail -1)
    echo "{\"impl\": \"$impl\", \"T\": $T, \"r\": $r}" >> $out
  done
done
cat $out
for T in 0 2; do
GCK_REPLAY_IMPL=b GCK_REPLAY_TMA=$T timeout 600 ncu --set full --import-source on --clock-control none -k regex:replay -s 2 -c 1 \
   -o gpurun_out/replay_v7b$T -f python scripts/microbench_replay.py > gpurun_out/ncu_replay_v7b$T.log 2>&1; echo "ncu rc=$?"
done
