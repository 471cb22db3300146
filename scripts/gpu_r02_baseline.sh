#!/bin/bash
# Round-2 baseline on this pod: GPU tests, smoke, default bench, replay microbench.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -5 | tee gpurun_out/r02a_gpu_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1 | tee gpurun_out/r02a_smoke.txt
timeout 900 python bench.py > gpurun_out/r02a_bench_default.json 2> gpurun_out/r02a_bench_default.err; tail -c 400 gpurun_out/r02a_bench_default.json
timeout 600 python scripts/microbench_replay.py > gpurun_out/r02a_microbench_replay.json 2>&1; cat gpurun_out/r02a_microbench_replay.json
nproc; free -g | head -2
