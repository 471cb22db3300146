#!/bin/bash
# Round-1 follow-up: new/changed GPU tests, smoke on the TMA kernel, box probe, TSan on the GPU session paths.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests -q -m gpu -k "multi_shard or e2e or K or session_staged" 2>&1 | tail -3
bash scripts/probe_box.sh > gpurun_out/box_probe.txt 2>&1
bash scripts/build_tsan.sh > /dev/null 2>&1 && \
  GCK_LIB_PATH=build/tsan/libgockpt_tsan.so LD_PRELOAD=$(gcc -print-file-name=libtsan.so) \
  TSAN_OPTIONS="halt_on_error=0 report_signal_unsafe=0 log_path=gpurun_out/tsan" \
  timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu \
  -k "eager or interleaved or multi_shard or automatic or drain_failure or gpu_replay_finalize" > gpurun_out/tsan_pytest.log 2>&1
tail -3 gpurun_out/tsan_pytest.log; ls gpurun_out | head -30
