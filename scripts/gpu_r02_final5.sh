#!/bin/bash
# Round-2 re-validation of the committed tree on a fresh box: the full GPU suite, smoke(), the
# default bench line, the reference arm with the driver's flags, and the replay microbench.
mkdir -p gpurun_out/fin5
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 2700 python -m pytest tests -q -m gpu 2>&1 | tail -6 | tee gpurun_out/fin5/r02_gpu_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1 | tee -a gpurun_out/fin5/r02_gpu_tests.txt
timeout 900 python bench.py > gpurun_out/fin5/r02_bench_default.json 2> gpurun_out/fin5/r02_bench_default.err
tail -c 300 gpurun_out/fin5/r02_bench_default.json
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/fin5/r02_bench_reference.json 2> gpurun_out/fin5/r02_bench_reference.err
tail -c 300 gpurun_out/fin5/r02_bench_reference.json
out=gpurun_out/fin5/r02_replay_final.jsonl; : > $out
for nk in "124439808 8" "124439808 4" "124439808 16" "842301952 8" "842301952 4"; do
  set -- $nk
  echo "{\"impl\": \"t\", \"r\": $(GCK_N=$1 GCK_K=$2 timeout 300 python scripts/microbench_replay.py 2>&1 | tail -1)}" >> $out
done
cat $out
