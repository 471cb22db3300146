#!/bin/bash
# BASELINE config 4 at 2 ranks with the SURVEY's long step (4x4096 tokens per rank, ~1 s steps): the
# regime where a 13B/2 rank's per-step transfer (up to 2n = 13 GB of gradient) fits in one step.
mkdir -p gpurun_out/cfg
python -c "import __graft_entry__ as g; g.build()" || exit 1
run() {
  local name=$1; shift
  timeout 2400 python bench.py "$@" --step-log gpurun_out/cfg/$name.steps.jsonl > gpurun_out/cfg/$name.json 2> gpurun_out/cfg/$name.err
  echo "$name rc=$? $(tail -c 300 gpurun_out/cfg/$name.json | head -c 300)"
}
run c4_13b_r2_t16k_k2_ring1 --model llama2-13b --shard-of 2 --tokens 16384 --K 2 --ring-slots 1 --interval 12 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline
run c4_13b_r2_t16k_k3_ring1 --model llama2-13b --shard-of 2 --tokens 16384 --K 3 --ring-slots 1 --interval 12 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline
run c4_13b_r2_t16k_k4_ring1 --model llama2-13b --shard-of 2 --tokens 16384 --K 4 --ring-slots 1 --interval 12 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline
run c4_13b_r2_t16k_k16_stream4 --model llama2-13b --shard-of 2 --tokens 16384 --K 16 --replay-mode stream --stream-buffers 4 --interval 20 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline
bash scripts/sanitize.sh > gpurun_out/r02_sanitize.txt 2>&1; grep -E "==|rc=|ERROR SUMMARY|RACECHECK SUMMARY" gpurun_out/r02_sanitize.txt
