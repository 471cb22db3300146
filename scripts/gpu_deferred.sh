#!/bin/bash
# NEXT-2 replay-on-restore: GPU tests of the deferred mode, then persist/restore cost per mode.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "deferred or persist" 2>&1 | tail -5 | tee gpurun_out/deferred_tests.txt
for n in 124439808 842301952; do
  for mode in host gpu deferred; do
    timeout 600 python scripts/bench_persist.py --n $n --K 8 --replay-mode $mode --threads 16 >> gpurun_out/persist_modes.jsonl 2>> gpurun_out/persist_modes.err
  done
done
cat gpurun_out/persist_modes.jsonl; tail -5 gpurun_out/persist_modes.err
