#!/bin/bash
# The round's GPU evidence in one call: tests, smoke, bench (default), ncu full of the fused
# kernel, and the launch list of a short bench run.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -c 3000 gpurun_out/bench_default.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.json 2>&1; tail -c 600 gpurun_out/bench_reference.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_adamw_pack -s 2 -c 3 \
    -o gpurun_out/fused -f python scripts/profile_fused.py > gpurun_out/ncu_full.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --interval 10 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/launches_bench.log 2>&1
ls -la gpurun_out
