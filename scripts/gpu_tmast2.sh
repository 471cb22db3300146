#!/bin/bash
# Bulk-store variant, round 2: output-ring depth sweep, then the live bench roofline (alternating impls).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
for gemm in 0 1; do
  GCK_MB_GEMM=$gemm timeout 300 python scripts/microbench_fused.py | sed "s/^/auto  gemm=$gemm /"
  for cfg in 3,3,16 3,4,16 3,5,16 4,4,16 2,4,16; do
    GCK_MB_GEMM=$gemm GCK_FUSED_IMPL=x GCK_TMAST_CFG=$cfg timeout 300 python scripts/microbench_fused.py | sed "s/^/x $cfg gemm=$gemm /"
  done
done 2>&1 | python -c "
import sys, json
for line in sys.stdin:
    head, _, js = line.partition('{')
    try: d = json.loads('{' + js)
    except Exception: print(line.rstrip()); continue
    print(head, 'plain %.0f GB/s  session %.0f GB/s' % (d['plain_gbs'], d['session_gbs']))" | tee gpurun_out/tmast2_mb.txt
for rep in 1 2; do for impl in auto x; do
  GCK_FUSED_IMPL=$impl timeout 900 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench2_impl_$impl.json 2> gpurun_out/bench2_impl_$impl.err
  python -c "
import json; d=json.loads(open('gpurun_out/bench2_impl_$impl.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$impl rep $rep', 'plain frac %.4f achieved %.0f' % (r['frac'], r['achieved']), 'session frac %.4f' % r['session_launches']['frac'], 'value %.0f' % d['value'], 'ratio %.4f' % d['ckpt_free']['throughput_ratio'], 'sm_mhz', d['clocks']['sm_mhz'])"
done; done 2>&1 | tee gpurun_out/tmast2_bench.txt
