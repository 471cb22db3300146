#!/bin/bash
# Host-code data-race checking (SURVEY §4.2 T0 "TSan builds of L1"): libgockpt with -fsanitize=thread on
# the C++ sources (kernels unchanged); run the threaded host paths (replay pool, persist writers) under it:
#   bash scripts/build_tsan.sh && GCK_LIB_PATH=build/tsan/libgockpt_tsan.so LD_PRELOAD=$(gcc -print-file-name=libtsan.so) \
#     TSAN_OPTIONS=halt_on_error=1 python -m pytest tests -m "not gpu" -k "lib_cpu or persist or property"
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUT=$ROOT/build/tsan
mkdir -p $OUT
CU=${CUDA_HOME:-/usr/local/cuda}
INC="-I $ROOT/include -I $ROOT/paper_2511_07035_b200/csrc -I $CU/include"
SAN="-fsanitize=thread -fno-omit-frame-pointer -g -O1"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC $INC -c $ROOT/paper_2511_07035_b200/csrc/kernels.cu -o $OUT/kernels.o
g++ -std=c++17 -fPIC $SAN $INC -c $ROOT/paper_2511_07035_b200/csrc/gockpt_runtime.cpp -o $OUT/runtime.o
g++ -std=c++17 -fPIC $SAN -ffp-contract=off -fno-math-errno $INC -c $ROOT/paper_2511_07035_b200/csrc/replay_host.cpp -o $OUT/replay_host.o
g++ -std=c++17 -fPIC $SAN $INC -c $ROOT/paper_2511_07035_b200/csrc/persist.cpp -o $OUT/persist.o
g++ -std=c++17 -fPIC $SAN $INC -c $ROOT/paper_2511_07035_b200/csrc/model.cpp -o $OUT/model.o
g++ -shared -fsanitize=thread -o $OUT/libgockpt_tsan.so $OUT/*.o -L $CU/lib64 -lcudart_static -lpthread -lz -ldl -lrt
echo $OUT/libgockpt_tsan.so
