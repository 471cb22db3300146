#!/bin/bash
# Final round-2 state: full GPU suite + smoke, TSan on the threaded session paths, default bench, the
# reference arm, 13B/4 K=8/16 with the folded verification.
mkdir -p gpurun_out/fin gpurun_out/cfg
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 2400 python -m pytest tests -q -m gpu 2>&1 | tail -4 | tee gpurun_out/fin/r02_gpu_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1 | tee -a gpurun_out/fin/r02_gpu_tests.txt
timeout 900 python bench.py --step-log gpurun_out/fin/r02_steps_gpt2.jsonl > gpurun_out/fin/r02_bench_default.json 2> gpurun_out/fin/r02_bench_default.err; tail -c 300 gpurun_out/fin/r02_bench_default.json
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/fin/r02_bench_reference.json 2>&1; tail -c 200 gpurun_out/fin/r02_bench_reference.json
for K in 8 16; do
  timeout 1500 python bench.py --model llama2-13b --shard-of 4 --K $K --interval 20 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline \
     --step-log gpurun_out/cfg/c4_13b_r4_k${K}_fold.steps.jsonl > gpurun_out/cfg/c4_13b_r4_k${K}_fold.json 2> gpurun_out/cfg/c4_13b_r4_k${K}_fold.err
  tail -c 200 gpurun_out/cfg/c4_13b_r4_k${K}_fold.json
done
bash scripts/build_tsan.sh > /dev/null 2>&1 && \
  GCK_LIB_PATH=build/tsan/libgockpt_tsan.so LD_PRELOAD=$(gcc -print-file-name=libtsan.so) \
  TSAN_OPTIONS="halt_on_error=0 report_signal_unsafe=0 log_path=gpurun_out/fin/tsan" \
  timeout 1500 python -m pytest tests/test_gpu_faults.py tests/test_gpu_parity.py -q -m gpu \
  -k "stream or deferred or eager or drain_failure or checkpointed or dropped or flipped or voided" > gpurun_out/fin/tsan_pytest.log 2>&1
tail -2 gpurun_out/fin/tsan_pytest.log; ls gpurun_out/fin | grep tsan | head; grep -l "WARNING: ThreadSanitizer" gpurun_out/fin/tsan* 2>/dev/null | head
