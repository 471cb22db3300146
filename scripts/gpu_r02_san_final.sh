#!/bin/bash
# compute-sanitizer on the final kernels (folded verification in the bulk-store fused kernel), plus the
# balanced plan through the same session script.
python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out/san
for tool in memcheck racecheck synccheck; do
  echo "== $tool"
  timeout 900 compute-sanitizer --tool $tool --target-processes all --kernel-name kns=gck \
      python scripts/sanitize_session.py > gpurun_out/san/sanitize_$tool.log 2>&1
  echo "rc=$?"; tail -3 gpurun_out/san/sanitize_$tool.log
done
echo "== memcheck, n = 1,000,003 (ragged tail through the folded checksum)"
GCK_N=1000003 timeout 900 compute-sanitizer --tool memcheck --target-processes all --kernel-name kns=gck \
    python scripts/sanitize_session.py > gpurun_out/san/sanitize_memcheck_1m.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/san/sanitize_memcheck_1m.log
