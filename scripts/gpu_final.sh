#!/bin/bash
# Final evidence pass: tests, smoke, default bench, kernel/replay microbenches, host replay scaling.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -c 400 gpurun_out/bench_default.json
timeout 600 python scripts/microbench_fused.py > gpurun_out/microbench_fused.json; cat gpurun_out/microbench_fused.json
timeout 600 python scripts/microbench_replay.py > gpurun_out/microbench_replay.json; cat gpurun_out/microbench_replay.json
timeout 900 python scripts/bench_host_replay.py > gpurun_out/host_replay.json; cat gpurun_out/host_replay.json
