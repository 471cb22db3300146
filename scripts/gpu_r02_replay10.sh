#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
out=gpurun_out/r02_replay10.jsonl; : > $out
for rep in 1 2; do
for c in 0 1; do
  for nk in "124439808 8" "124439808 4" "842301952 8"; do
    set -- $nk
    echo "{\"coalesced\": $c, \"r\": $(GCK_REPLAY_COALESCED=$c GCK_N=$1 GCK_K=$2 timeout 300 python scripts/microbench_replay.py 2>&1 | tail -1)}" >> $out
  done
done
done
cat $out
GCK_REPLAY_COALESCED=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:replay -s 2 -c 1 \
   -o gpurun_out/replay_coal -f python scripts/microbench_replay.py > gpurun_out/ncu_replay_coal.log 2>&1; echo "ncu rc=$?"
GCK_REPLAY_COALESCED=1 timeout 900 python -m pytest tests/test_gpu_guard.py tests/test_gpu_fullsize.py -q -m gpu 2>&1 | tail -3
