#!/bin/bash
# Cost of the folded verification checksums inside the host replay, on the GPU box's host CPU.
mkdir -p gpurun_out/hs
g++ -O3 -std=c++17 -ffp-contract=off -fno-math-errno -Iinclude -Ipaper_2511_07035_b200/csrc -I/usr/local/cuda/include \
    scripts/c/replay_sums_bench.cpp paper_2511_07035_b200/csrc/replay_host.cpp -o /tmp/rsb -lpthread || exit 1
for nk in "124439808 8" "124439808 16" "842301952 8"; do
  set -- $nk
  /tmp/rsb $1 $2 0 | tee -a gpurun_out/hs/hostsums.txt
  GCK_EVICT_BYTES=0 /tmp/rsb $1 $2 0 | sed 's/^/evict-off /' | tee -a gpurun_out/hs/hostsums.txt
done
