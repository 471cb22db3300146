#!/bin/bash
# Streaming host replay + replay-on-restore: GPU tests, then the default bench per replay mode.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "stream or deferred or drain_failure or checkpointed or persist" 2>&1 | tail -5 | tee gpurun_out/stream_tests.txt
for mode in host stream; do
  timeout 900 python bench.py --replay-mode $mode --no-cpu-baseline > gpurun_out/bench_replay_$mode.json 2> gpurun_out/bench_replay_$mode.err
  tail -c 400 gpurun_out/bench_replay_$mode.err
done
timeout 900 python bench.py --replay-mode stream --stream-buffers 3 --no-cpu-baseline > gpurun_out/bench_replay_stream3.json 2> gpurun_out/bench_replay_stream3.err
timeout 900 python bench.py --replay-mode deferred --no-cpu-baseline > gpurun_out/bench_replay_deferred.json 2> gpurun_out/bench_replay_deferred.err
for f in gpurun_out/bench_replay_*.json; do echo $f; python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(json.dumps({k: d[k] for k in ('value','stall','d2h','replay','ckpt_free')}))"; done
