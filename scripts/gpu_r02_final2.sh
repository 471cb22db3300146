#!/bin/bash
# After folding the drain verification into the replay: fault/parity tests of that path, default bench
# (verification on/off), CUPTI timeline at the bench's interval, 13B/2 long-step configs, sanitizers.
mkdir -p gpurun_out/ev2
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1800 python -m pytest tests/test_gpu_faults.py tests/test_gpu_parity.py tests/test_gpu_guard.py -q -m gpu 2>&1 | tail -3 | tee gpurun_out/ev2/tests.txt
timeout 900 python bench.py --step-log gpurun_out/ev2/r02_steps_gpt2.jsonl > gpurun_out/ev2/r02_bench_default.json 2> gpurun_out/ev2/r02_bench_default.err; tail -c 300 gpurun_out/ev2/r02_bench_default.json
timeout 900 python bench.py --verify-drain 0 > gpurun_out/ev2/r02_bench_noverify.json 2> gpurun_out/ev2/r02_bench_noverify.err; tail -c 200 gpurun_out/ev2/r02_bench_noverify.json
timeout 900 python scripts/timeline.py --interval 50 --out gpurun_out/ev2/r02_timeline > gpurun_out/ev2/timeline.log 2>&1; tail -3 gpurun_out/ev2/timeline.log
bash scripts/gpu_r02_configs_long.sh
