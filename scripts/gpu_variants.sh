#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for v in ${VARIANTS:-"simple 0" "tma 3,2" "tma 5,1" "tma 6,1" "tma 7,1" "tma 8,1"}; do
  set -- $v
  GCK_FUSED_IMPL=$1 GCK_TMA_CFG=$2 timeout 300 python scripts/microbench_fused.py
done
