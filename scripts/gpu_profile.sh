#!/bin/bash
# One gpurun call: full ncu capture of fused_adamw_pack + the bench launch list.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
ncu --set full --clock-control none --import-source on -k regex:fused_adamw_pack -s 2 -c 3 \
    -o gpurun_out/fused -f python scripts/profile_fused.py > gpurun_out/ncu_full.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --interval 10 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/launches_bench.log 2>&1
tail -3 gpurun_out/ncu_full.log gpurun_out/launches_bench.log
