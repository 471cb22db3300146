#!/bin/bash
# Streaming replay with batched slice application: GPU tests, then 13B/K=16 and GPT-2/K=8 against batch.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "stream or drain_failure" 2>&1 | tail -2 | tee gpurun_out/streamb_tests.txt
bash scripts/gpu_stream13b.sh 2>&1 | tail -2
for B in 2 4; do
  timeout 900 python bench.py --model llama2-13b --shard-of 8 --K 16 --interval 24 --steps 2 --warmup 3 \
      --replay-mode stream --stream-buffers $B --no-e2e --no-cpu-baseline > gpurun_out/stream13b_B$B.json 2> /dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/stream13b_B$B.json').read().strip().splitlines()[-1]); s=d['stall']; r=d['replay']
print('stream B=$B', 'ratio %.4f' % d['ckpt_free']['throughput_ratio'], 'delta/session step %.2f ms (%.2f%%)' % (s['delta_ms_per_session_step_mean'], 100*s['delta_frac_of_step']), 'D2H %.1f GB/s' % d['d2h']['gbs'], 'replay arithmetic %.0f ms' % r['host_ms_last_session'], 'finalize wait %.0f ms' % r['finalize_wait_ms_last'], 'swait %.0f ms' % (r.get('stream_wait_ms_last') or 0))"
done 2>&1 | tee -a gpurun_out/stream13b.txt
for mode in host stream; do
  timeout 900 python bench.py --replay-mode $mode --no-cpu-baseline --no-e2e > gpurun_out/streamb_gpt2_$mode.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/streamb_gpt2_$mode.json').read().strip().splitlines()[-1]); s=d['stall']; r=d['replay']
print('gpt2 $mode', 'ratio %.4f' % d['ckpt_free']['throughput_ratio'], 'delta/session step %.3f ms' % s['delta_ms_per_session_step_mean'], 'D2H %.1f GB/s' % d['d2h']['gbs'], 'replay arithmetic %.0f ms' % r['host_ms_last_session'], 'swait %.0f ms' % (r.get('stream_wait_ms_last') or 0))"
done 2>&1 | tee gpurun_out/streamb_gpt2.txt
