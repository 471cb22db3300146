#!/bin/bash
# Streaming vs batch host replay at the K=16 point of BASELINE config 4 (13B rank-of-8 shard), where the
# streaming arena (12n + 4n) is smallest relative to the batch one (12n + 15n).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
for mode in host stream; do
  timeout 900 python bench.py --model llama2-13b --shard-of 8 --K 16 --interval 24 --steps 2 --warmup 3 \
      --replay-mode $mode --no-e2e --no-cpu-baseline > gpurun_out/stream13b_$mode.json 2> gpurun_out/stream13b_$mode.err
  python -c "
import json; d=json.loads(open('gpurun_out/stream13b_$mode.json').read().strip().splitlines()[-1]); s=d['stall']; r=d['replay']
print('$mode', 'ratio %.4f' % d['ckpt_free']['throughput_ratio'], 'delta/session step %.2f ms (%.2f%%)' % (s['delta_ms_per_session_step_mean'], 100*s['delta_frac_of_step']), 'D2H %.1f GB/s' % d['d2h']['gbs'], 'replay arithmetic %.0f ms' % r['host_ms_last_session'], 'finalize wait %.0f ms' % r['finalize_wait_ms_last'], 'swait %.0f ms' % (r.get('stream_wait_ms_last') or 0), 'HBM %.1f%%' % (100*d['roofline']['frac']))"
done 2>&1 | tee gpurun_out/stream13b.txt
