#!/bin/bash
# VARIANTS="simple:0 tma:6,1,8 ..." GEMMS="0 1" TESTS=1
python -c "import __graft_entry__ as g; g.build()" || exit 1
[ -n "$TESTS" ] && timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for gemm in ${GEMMS:-0 1}; do
for v in ${VARIANTS:-simple:0 tma:6,1,8 tma:6,1,16 tma:4,1,16 tma:8,1,16 tma:3,2,16 tma:3,2,8}; do
  impl=${v%%:*}; cfg=${v#*:}
  GCK_MB_GEMM=$gemm GCK_FUSED_IMPL=$impl GCK_TMA_CFG=$cfg timeout 300 python scripts/microbench_fused.py | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['impl'], d['cfg'], 'gemm ' if d['gemm_burst'] else 'clean', 'plain %.0f us %.0f GB/s | session %.0f us %.0f GB/s' % (d['plain_us_mean'], d['plain_gbs'], d['session_us_mean'], d['session_gbs']))"
done; done
