#!/bin/bash
# Refresh the round's evidence with the current kernels: tests, smoke, bench (+ reference arm),
# ncu --set full of the fused kernel, microbenches.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -1
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_adamw_pack -s 2 -c 3 \
    -o gpurun_out/fused -f python scripts/profile_fused.py > gpurun_out/ncu_full.log 2>&1
timeout 600 python scripts/microbench_fused.py > gpurun_out/microbench_fused.json
timeout 600 python scripts/microbench_replay.py > gpurun_out/microbench_replay.json
timeout 900 python scripts/bench_host_replay.py > gpurun_out/host_replay.json
ls gpurun_out
