#!/bin/bash
# Streaming replay (per-slice application): slice-buffer count B at 13B rank-of-8, K=16.
python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out
for B in 2 4 8; do
  timeout 900 python bench.py --model llama2-13b --shard-of 8 --K 16 --interval 24 --steps 2 --warmup 3 \
      --replay-mode stream --stream-buffers $B --no-e2e --no-cpu-baseline > gpurun_out/streamB$B.json 2> /dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/streamB$B.json').read().strip().splitlines()[-1]); s=d['stall']; r=d['replay']
print('stream B=$B', 'ratio %.4f' % d['ckpt_free']['throughput_ratio'], 'delta/session step %.2f ms (%.2f%%)' % (s['delta_ms_per_session_step_mean'], 100*s['delta_frac_of_step']), 'D2H %.1f GB/s' % d['d2h']['gbs'], 'replay arithmetic %.0f ms' % r['host_ms_last_session'], 'finalize wait %.0f ms' % r['finalize_wait_ms_last'], 'swait %.0f ms' % (r.get('stream_wait_ms_last') or 0))"
done 2>&1 | tee gpurun_out/streamB.txt
