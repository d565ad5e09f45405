#!/bin/bash
# Build an A/B variant of libmdg.so with extra nvcc flags: tools/build_variant.sh NAME "-DFOO=1"
set -e
NAME=$1; FLAGS=$2
P=paper_1911_08963_b200
OUT=tools/variants/build_$NAME
mkdir -p $OUT tools/variants
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude"
$NV $FLAGS -c $P/csrc/engine.cu -o $OUT/engine.o
$NV $FLAGS -c $P/csrc/gsearch.cu -o $OUT/gsearch.o
g++ -std=c++17 -O3 -fPIC -Iinclude -I/usr/local/cuda/include -c $P/csrc/host.cpp -o $OUT/host.o
g++ -std=c++17 -O3 -fPIC -Iinclude -I/usr/local/cuda/include -c $P/csrc/capi.cpp -o $OUT/capi.o
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o tools/variants/libmdg_$NAME.so $OUT/*.o -ldl -lpthread
echo built tools/variants/libmdg_$NAME.so
