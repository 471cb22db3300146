#!/bin/bash
# Final-tree evidence: full GPU suite + smoke, default bench, reference arm, replay microbench,
# ncu --set full of the fused kernel + a bench launch list, and the config lines (C1, C3, C4 13B/4).
mkdir -p gpurun_out/fin6 gpurun_out/fin6/cfg
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 2700 python -m pytest tests -q -m gpu 2>&1 | tail -6 | tee gpurun_out/fin6/r02_gpu_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1 | tee -a gpurun_out/fin6/r02_gpu_tests.txt
timeout 900 python bench.py > gpurun_out/fin6/r02_bench_default.json 2> gpurun_out/fin6/r02_bench_default.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/fin6/r02_bench_reference.json 2> gpurun_out/fin6/r02_bench_reference.err
out=gpurun_out/fin6/r02_replay_final.jsonl; : > $out
for nk in "124439808 8" "124439808 4" "124439808 16" "842301952 8" "842301952 4"; do
  set -- $nk
  echo "{\"impl\": \"t\", \"r\": $(GCK_N=$1 GCK_K=$2 timeout 300 python scripts/microbench_replay.py 2>&1 | tail -1)}" >> $out
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_adamw_pack -s 2 -c 3 \
    -o gpurun_out/fin6/fused -f python scripts/profile_fused.py > gpurun_out/fin6/ncu_full.log 2>&1; echo "ncu full rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin6/launches.csv \
    python bench.py --interval 10 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/fin6/launches_bench.log 2>&1; echo "ncu list rc=$?"
run() {  # name, args...
  local name=$1; shift
  timeout 1800 python bench.py "$@" --step-log gpurun_out/fin6/cfg/$name.steps.jsonl > gpurun_out/fin6/cfg/$name.json 2> gpurun_out/fin6/cfg/$name.err
  echo "$name rc=$?"
}
run c1_spin1 --model flat-1m --K 4 --interval 20 --steps 5 --warmup 3 --spin-ms 1
run c1_spin0 --model flat-1m --K 4 --interval 20 --steps 5 --warmup 3 --spin-ms 0
run c3_7b_r8_i100 --model llama2-7b --shard-of 8 --K 8 --interval 100 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline
for K in 2 4 8 16; do
  run c4_13b_r4_i50_k$K --model llama2-13b --shard-of 4 --K $K --interval 50 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline
done
for K in 4 6 8; do
  run c4_13b_r4_i50_k${K}_balanced --model llama2-13b --shard-of 4 --K $K --interval 50 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --plan balanced
done
run c4_13b_r4_k16 --model llama2-13b --shard-of 4 --K 16 --interval 20 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline
