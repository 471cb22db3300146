#!/bin/bash
# Final-tree refresh of BASELINE config 4 at 2 ranks (n_r = 6.5e9 > 2^32): the short-step lines
# (R = 1 ring, direct, streaming) and the SURVEY's long-step regime, plus the balanced plan.
mkdir -p gpurun_out/fin6/cfg
python -c "import __graft_entry__ as g; g.build()" || exit 1
run() {  # name, args...
  local name=$1; shift
  timeout 2400 python bench.py "$@" --step-log gpurun_out/fin6/cfg/$name.steps.jsonl > gpurun_out/fin6/cfg/$name.json 2> gpurun_out/fin6/cfg/$name.err
  echo "$name rc=$?"
}
C="--model llama2-13b --shard-of 2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
run c4_13b_r2_k2_ring1 $C --K 2 --ring-slots 1 --interval 20
run c4_13b_r2_k3_ring1 $C --K 3 --ring-slots 1 --interval 20
run c4_13b_r2_k2_direct $C --K 2 --staging direct --interval 20
run c4_13b_r2_k3_direct $C --K 3 --staging direct --interval 20
run c4_13b_r2_k16_stream4 $C --K 16 --replay-mode stream --stream-buffers 4 --interval 20
run c4_13b_r2_k16_stream4_balanced $C --K 16 --replay-mode stream --stream-buffers 4 --interval 20 --plan balanced
run c4_13b_r2_t16k_k2_ring1 $C --tokens 16384 --K 2 --ring-slots 1 --interval 12
run c4_13b_r2_t16k_k3_ring1 $C --tokens 16384 --K 3 --ring-slots 1 --interval 12
run c4_13b_r2_t16k_k4_ring1 $C --tokens 16384 --K 4 --ring-slots 1 --interval 12
run c4_13b_r2_t16k_k16_stream4 $C --tokens 16384 --K 16 --replay-mode stream --stream-buffers 4 --interval 20
free -g | head -2
