#!/bin/bash
# Final round-1 evidence with the bulk-store default kernel: tests, smoke, sanitizers, TSan (stream/deferred),
# default bench, reference arm, ncu --set full of the fused kernel, short launch list, microbenches.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -3 | tee gpurun_out/final_gpu_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1 | tee gpurun_out/final_smoke.txt
timeout 900 python bench.py > gpurun_out/final_bench_default.json 2> gpurun_out/final_bench_default.err; tail -c 600 gpurun_out/final_bench_default.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final_bench_reference.json 2>&1; tail -c 300 gpurun_out/final_bench_reference.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_adamw_pack -s 2 -c 3 \
    -o gpurun_out/fused_final -f python scripts/profile_fused.py > gpurun_out/ncu_full_final.log 2>&1; echo "ncu full rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv \
    python bench.py --interval 10 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/launches_final_bench.log 2>&1; echo "ncu list rc=$?"
timeout 600 python scripts/microbench_fused.py > gpurun_out/final_microbench_fused.json; cat gpurun_out/final_microbench_fused.json
GCK_MB_GEMM=1 timeout 600 python scripts/microbench_fused.py > gpurun_out/final_microbench_fused_gemm.json; cat gpurun_out/final_microbench_fused_gemm.json
bash scripts/sanitize.sh > gpurun_out/final_sanitize.txt 2>&1; cat gpurun_out/final_sanitize.txt | grep -E "==|rc=|ERROR SUMMARY|RACECHECK SUMMARY"
bash scripts/build_tsan.sh > /dev/null 2>&1 && \
  GCK_LIB_PATH=build/tsan/libgockpt_tsan.so LD_PRELOAD=$(gcc -print-file-name=libtsan.so) \
  TSAN_OPTIONS="halt_on_error=0 report_signal_unsafe=0 log_path=gpurun_out/tsan_final" \
  timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu \
  -k "stream or deferred or eager or drain_failure or checkpointed" > gpurun_out/final_tsan_pytest.log 2>&1
tail -2 gpurun_out/final_tsan_pytest.log; ls gpurun_out/ | grep tsan_final | head; grep -l "WARNING: ThreadSanitizer" gpurun_out/tsan_final* 2>/dev/null | head
