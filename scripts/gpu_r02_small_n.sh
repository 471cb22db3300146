#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
out=gpurun_out/r02_small_n.jsonl; : > $out
for n in 262144 1048576 4194304 16777216; do
  for impl in auto s t; do
    echo "{\"n\": $n, \"impl\": \"$impl\", \"r\": $(GCK_N=$n GCK_FUSED_IMPL=$impl timeout 300 python scripts/microbench_fused.py 2>&1 | tail -1)}" >> $out
  done
done
cat $out
