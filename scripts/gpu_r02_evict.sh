#!/bin/bash
# Tail eviction of the host passes' cache lines (evict_budget): small-session drains, C1 bench lines,
# host replay cost with and without it, and the default bench line.
mkdir -p gpurun_out/evict
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 300 python scripts/diag_small_drain2.py sync b2b > gpurun_out/evict/small2.jsonl 2>&1
GCK_EVICT_BYTES=0 timeout 300 python scripts/diag_small_drain2.py sync b2b > gpurun_out/evict/small2_off.jsonl 2>&1
cat > /tmp/hr.py <<'PY'
import json, os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
import gockpt_inputs as gi
import paper_2511_07035_b200 as G
n, K = int(sys.argv[1]), int(sys.argv[2])
parts = G.plan_parts(n, K, 1024)
recs = [G.make_step_record(0.9, 0.999, 1e-8, 0.01, 100 + i, 3e-4) for i in range(1, K + 1)]
base = gi.warm_state(1, n)
glog = [gi.grad_bits(1, 101 + i, parts[i][1]) for i in range(K - 1)]
ts = []
for r in range(6):
    p, m, v = (x.copy() for x in base)
    t = time.perf_counter(); G.replay_host(recs, parts, p, m, v, glog); ts.append((time.perf_counter() - t) * 1e3)
print(json.dumps({"n": n, "K": K, "evict": os.environ.get("GCK_EVICT_BYTES", "default"), "ms": sorted(ts[1:])}))
PY
for nk in "1048576 4" "124439808 8"; do
  set -- $nk
  timeout 300 python /tmp/hr.py $1 $2 >> gpurun_out/evict/host_replay.jsonl 2>&1
  GCK_EVICT_BYTES=0 timeout 300 python /tmp/hr.py $1 $2 >> gpurun_out/evict/host_replay.jsonl 2>&1
done
run() {  # name, args...
  local name=$1; shift
  timeout 900 python bench.py "$@" --step-log gpurun_out/evict/$name.steps.jsonl > gpurun_out/evict/$name.json 2> gpurun_out/evict/$name.err
  echo "$name rc=$?"
}
run c1_spin1 --model flat-1m --K 4 --interval 20 --steps 5 --warmup 3 --spin-ms 1
run c1_spin0 --model flat-1m --K 4 --interval 20 --steps 5 --warmup 3 --spin-ms 0
run default
cat gpurun_out/evict/host_replay.jsonl
