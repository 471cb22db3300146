#!/bin/bash
# Refresh every measured table with the current code in one call: configs 3-4 (K sweep, 7B rank shard),
# NEXT-3 schemes, the 1000-step long run, fused/replay microbenches, host replay scaling.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
bash scripts/k_sweep.sh 2> gpurun_out/k_sweep.err
bash scripts/scheme_compare.sh > gpurun_out/schemes.txt 2>&1
timeout 1200 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_long.json 2> gpurun_out/bench_long.err
timeout 600 python scripts/microbench_fused.py > gpurun_out/microbench_fused.json
timeout 600 python scripts/microbench_replay.py > gpurun_out/microbench_replay.json
timeout 900 python scripts/bench_host_replay.py > gpurun_out/host_replay.json
wc -l gpurun_out/k_sweep.jsonl gpurun_out/schemes.jsonl; tail -c 300 gpurun_out/bench_long.json; cat gpurun_out/microbench_fused.json
