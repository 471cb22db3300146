#!/bin/bash
# initcheck controls for the checksum kernel's reads of bulk-copy-written slot bytes; the NCCL path as a
# process group of one; 13B rank-of-4 K=8/16 with the verification folded into the replay.
mkdir -p gpurun_out/ctl
python -c "import __graft_entry__ as g; g.build()" || exit 1
GCK_FUSED_IMPL=s timeout 900 compute-sanitizer --tool initcheck --target-processes all --kernel-name kns=gck \
   python scripts/sanitize_session.py > gpurun_out/ctl/initcheck_stg.log 2>&1; echo "initcheck STG-store fused kernel rc=$?"; tail -2 gpurun_out/ctl/initcheck_stg.log
GCK_SANITIZE_VERIFY=0 timeout 900 compute-sanitizer --tool initcheck --target-processes all --kernel-name kns=gck \
   python scripts/sanitize_session.py > gpurun_out/ctl/initcheck_noverify.log 2>&1; echo "initcheck no verification rc=$?"; tail -2 gpurun_out/ctl/initcheck_noverify.log
timeout 1200 python -m pytest tests/test_gpu_dist_smoke.py -q -m gpu 2>&1 | tail -3 | tee gpurun_out/ctl/dist_tests.txt
for K in 8 16; do
  timeout 1500 python bench.py --model llama2-13b --shard-of 4 --K $K --interval 20 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline \
     --step-log gpurun_out/cfg/c4_13b_r4_k${K}_fold.steps.jsonl > gpurun_out/cfg/c4_13b_r4_k${K}_fold.json 2> gpurun_out/cfg/c4_13b_r4_k${K}_fold.err
  tail -c 200 gpurun_out/cfg/c4_13b_r4_k${K}_fold.json
done
