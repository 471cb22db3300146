#!/bin/bash
mkdir -p gpurun_out/q
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 python -m pytest tests/test_gpu_guard.py tests/test_gpu_dist_smoke.py -q -m gpu 2>&1 | tail -6 | tee gpurun_out/q/tests.txt
