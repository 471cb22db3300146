#!/bin/bash
mkdir -p gpurun_out/ctl
python -c "import __graft_entry__ as g; g.build()" || exit 1
MASTER_ADDR=127.0.0.1 MASTER_PORT=29533 WORLD_SIZE=1 RANK=0 LOCAL_RANK=0 timeout 300 python scripts/nccl_probe.py > gpurun_out/ctl/probe.out 2> gpurun_out/ctl/probe.err; echo "probe rc=$?"
grep -c "NCCL INFO" gpurun_out/ctl/probe.err gpurun_out/ctl/probe.out; tail -3 gpurun_out/ctl/probe.err
MASTER_ADDR=127.0.0.1 MASTER_PORT=29534 WORLD_SIZE=1 RANK=0 LOCAL_RANK=0 NCCL_DEBUG_FILE=/dev/stderr timeout 300 python scripts/nccl_probe.py > gpurun_out/ctl/probe2.out 2> gpurun_out/ctl/probe2.err; echo "probe2 rc=$?"
grep -c "NCCL INFO" gpurun_out/ctl/probe2.err gpurun_out/ctl/probe2.out
timeout 900 python -m pytest tests/test_gpu_dist_smoke.py -q -m gpu -k nccl -x 2>&1 | tail -30 > gpurun_out/ctl/nccl_test2.txt
