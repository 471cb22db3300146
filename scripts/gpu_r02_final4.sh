#!/bin/bash
mkdir -p gpurun_out/fin4
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 2400 python -m pytest tests -q -m gpu 2>&1 | tail -4 | tee gpurun_out/fin4/r02_gpu_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1 | tee -a gpurun_out/fin4/r02_gpu_tests.txt
timeout 900 python bench.py > gpurun_out/fin4/r02_bench_default.json 2> gpurun_out/fin4/r02_bench_default.err; tail -c 300 gpurun_out/fin4/r02_bench_default.json
timeout 900 python bench.py --replay-mode gpu > gpurun_out/fin4/r02_bench_gpu_replay.json 2> gpurun_out/fin4/r02_bench_gpu_replay.err; tail -c 200 gpurun_out/fin4/r02_bench_gpu_replay.json
