#!/bin/bash
# Host-code memory/UB checking: build libgockpt with -fsanitize=address,undefined on the C++ sources
# (kernels unchanged) and run the CPU test suite against it:
#   bash scripts/build_asan.sh && GCK_LIB_PATH=build/asan/libgockpt_asan.so \
#     LD_PRELOAD=$(gcc -print-file-name=libasan.so) ASAN_OPTIONS=detect_leaks=0,protect_shadow_gap=0 \
#     python -m pytest tests -m "not gpu" -k "lib_cpu or persist or property or analytic"
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUT=$ROOT/build/asan
mkdir -p $OUT
CU=${CUDA_HOME:-/usr/local/cuda}
INC="-I $ROOT/include -I $ROOT/paper_2511_07035_b200/csrc -I $CU/include"
SAN="-fsanitize=address,undefined -fno-omit-frame-pointer -g -O1"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC $INC -c $ROOT/paper_2511_07035_b200/csrc/kernels.cu -o $OUT/kernels.o
g++ -std=c++17 -fPIC $SAN $INC -c $ROOT/paper_2511_07035_b200/csrc/gockpt_runtime.cpp -o $OUT/runtime.o
g++ -std=c++17 -fPIC $SAN -ffp-contract=off -fno-math-errno $INC -c $ROOT/paper_2511_07035_b200/csrc/replay_host.cpp -o $OUT/replay_host.o
g++ -std=c++17 -fPIC $SAN $INC -c $ROOT/paper_2511_07035_b200/csrc/persist.cpp -o $OUT/persist.o
g++ -std=c++17 -fPIC $SAN $INC -c $ROOT/paper_2511_07035_b200/csrc/model.cpp -o $OUT/model.o
g++ -shared -fsanitize=address,undefined -o $OUT/libgockpt_asan.so $OUT/*.o -L $CU/lib64 -lcudart_static -lpthread -lz -ldl -lrt
echo $OUT/libgockpt_asan.so
