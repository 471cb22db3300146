#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
out=gpurun_out/r02_replay9.jsonl; : > $out
for rep in 1 2; do
for pf in 0 1 2; do
  for nk in "124439808 8" "124439808 4" "842301952 8"; do
    set -- $nk
    echo "{\"pref\": $pf, \"r\": $(GCK_REPLAY_PREF=$pf GCK_N=$1 GCK_K=$2 timeout 300 python scripts/microbench_replay.py 2>&1 | tail -1)}" >> $out
  done
done
done
cat $out
GCK_REPLAY_PREF=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:replay -s 2 -c 1 \
   -o gpurun_out/replay_pref1 -f python scripts/microbench_replay.py > gpurun_out/ncu_replay_pref1.log 2>&1; echo "ncu rc=$?"
