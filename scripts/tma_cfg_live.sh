#!/bin/bash
# Fused-kernel configuration under the LIVE bench (GEMM-heavy F/B between launches, power-capped clocks):
# roofline.frac of the plain and session launches per GCK_TMA_CFG (stages,CTAs/SM,consumer warps).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
OUT=gpurun_out/tma_cfg_live.jsonl
: > $OUT
for rep in 1 2; do
for cfg in 4,1,16 6,1,16 8,1,16 4,1,24 3,2,16 3,2,8; do
  GCK_TMA_CFG=$cfg timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline \
    | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print(json.dumps({'cfg':'$cfg','plain_frac':r['frac'],'plain_us':r['mean_launch_us'],'sess_frac':r['session_launches']['frac'],'sm_mhz':d['clocks']['sm_mhz'],'ratio':d['ckpt_free']['throughput_ratio']}))" >> $OUT
done; done
cat $OUT
