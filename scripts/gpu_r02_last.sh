#!/bin/bash
# Last evidence on the final tree: CUPTI overlap timeline and a 1000-step run (20 sessions).
mkdir -p gpurun_out/last
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python scripts/timeline.py --interval 50 --out gpurun_out/last/r02_timeline > gpurun_out/last/timeline.log 2>&1; tail -3 gpurun_out/last/timeline.log
timeout 1500 python bench.py --steps 20 --warmup 3 --step-log gpurun_out/last/r02_bench_long_20intervals.steps.jsonl \
    > gpurun_out/last/r02_bench_long_20intervals.json 2> gpurun_out/last/long.err
echo "long rc=$?"; tail -c 300 gpurun_out/last/r02_bench_long_20intervals.json
