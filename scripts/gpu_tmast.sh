#!/bin/bash
# The bulk-store variant of the fused kernel (GCK_FUSED_IMPL=x): parity under it, then speed vs the STG variant.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
GCK_FUSED_IMPL=x timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -m gpu -x 2>&1 | tail -4 | tee gpurun_out/tmast_tests.txt
for gemm in 0 1; do
  GCK_MB_GEMM=$gemm timeout 300 python scripts/microbench_fused.py | sed "s/^/auto  gemm=$gemm /"
  for cfg in 4,2,16 3,3,16 4,3,16 5,2,16 4,2,8; do
    GCK_MB_GEMM=$gemm GCK_FUSED_IMPL=x GCK_TMAST_CFG=$cfg timeout 300 python scripts/microbench_fused.py | sed "s/^/x $cfg gemm=$gemm /"
  done
done 2>&1 | tee gpurun_out/tmast_mb.txt
for impl in auto x; do
  GCK_FUSED_IMPL=$impl timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_impl_$impl.json 2> gpurun_out/bench_impl_$impl.err
  python -c "
import json; d=json.loads(open('gpurun_out/bench_impl_$impl.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$impl', 'plain frac %.4f achieved %.0f' % (r['frac'], r['achieved']), 'session frac %.4f' % r['session_launches']['frac'], 'value %.0f' % d['value'], 'sm_mhz', d['clocks']['sm_mhz'])"
done 2>&1 | tee gpurun_out/tmast_bench.txt
