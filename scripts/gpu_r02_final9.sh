#!/bin/bash
# Final tree with 128-thread replay CTAs: full GPU suite + smoke and the replay microbench.
mkdir -p gpurun_out/fin9
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -4 | tee gpurun_out/fin9/r02_gpu_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1 | tee -a gpurun_out/fin9/r02_gpu_tests.txt
out=gpurun_out/fin9/r02_replay_final.jsonl; : > $out
for nk in "124439808 8" "124439808 4" "124439808 16" "842301952 8" "842301952 4"; do
  set -- $nk
  echo "{\"impl\": \"t\", \"r\": $(GCK_N=$1 GCK_K=$2 timeout 300 python scripts/microbench_replay.py 2>&1 | tail -1)}" >> $out
done
cat $out
