#!/bin/bash
# The ncu launch list of the exact default bench command (B200_PROFILING.md: gpu__time_duration.sum,
# --clock-control none). Serialised and cold-cache: compare the kernels' SHARES of a step.
python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
timeout ${NCU_LIMIT:-2400} ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_default.csv \
    python bench.py > gpurun_out/launches_default_bench.log 2>&1
echo "ncu rc=$?"; ls -la gpurun_out/launches_default.csv; tail -c 300 gpurun_out/launches_default_bench.log
