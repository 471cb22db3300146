#!/bin/bash
# Round-2 evidence: default bench (+ step log), verification on/off, reference arm (the driver's command),
# CUPTI timeline, ncu --set full of the fused kernel, ncu launch list of a short bench, GPU tests + smoke.
mkdir -p gpurun_out/ev
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python bench.py --step-log gpurun_out/ev/r02_steps_gpt2.jsonl > gpurun_out/ev/r02_bench_default.json 2> gpurun_out/ev/r02_bench_default.err; tail -c 300 gpurun_out/ev/r02_bench_default.json
timeout 900 python bench.py --verify-drain 0 > gpurun_out/ev/r02_bench_noverify.json 2> gpurun_out/ev/r02_bench_noverify.err; tail -c 200 gpurun_out/ev/r02_bench_noverify.json
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ev/r02_bench_reference.json 2>&1; tail -c 300 gpurun_out/ev/r02_bench_reference.json
timeout 900 python scripts/timeline.py --out gpurun_out/ev/r02_timeline > gpurun_out/ev/timeline.log 2>&1; tail -3 gpurun_out/ev/timeline.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_adamw_pack -s 2 -c 3 \
    -o gpurun_out/ev/fused_r02 -f python scripts/profile_fused.py > gpurun_out/ev/ncu_full_fused.log 2>&1; echo "ncu full rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev/launches_r02.csv \
    python bench.py --interval 10 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ev/launches_bench.log 2>&1; echo "ncu list rc=$?"
for rep in 1 2; do
  timeout 900 python scripts/microbench_fused.py >> gpurun_out/ev/r02_microbench_fused.json 2>&1
  GCK_FUSED_GUARD=g timeout 900 python scripts/microbench_fused.py >> gpurun_out/ev/r02_microbench_fused_oldguard.json 2>&1
  GCK_MB_GEMM=1 timeout 900 python scripts/microbench_fused.py >> gpurun_out/ev/r02_microbench_fused_gemm.json 2>&1
  GCK_MB_GEMM=1 GCK_FUSED_GUARD=g timeout 900 python scripts/microbench_fused.py >> gpurun_out/ev/r02_microbench_fused_gemm_oldguard.json 2>&1
done
tail -c 300 gpurun_out/ev/r02_microbench_fused*.json
timeout 2400 python -m pytest tests -q -m gpu 2>&1 | tail -4 | tee gpurun_out/ev/r02_gpu_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1 | tee gpurun_out/ev/r02_smoke.txt
which nsys; ls /usr/local/cuda/bin | grep -i nsys
