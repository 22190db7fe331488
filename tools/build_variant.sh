#!/bin/bash
# Build a compile-time A/B variant of libprgpu into build/<name>.so (tool;
# select it with PRGPU_LIB=build/<name>.so, e.g. through tools/ab_env.py).
# Usage: tools/build_variant.sh <name> -DMACRO=value ...
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p build/$name
C=paper_2109_09527_b200/csrc
for f in api ingest preprocess iterate blocked shard multicast; do
  nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
       --expt-relaxed-constexpr "$@" -c $C/$f.cu -o build/$name/$f.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/$name.so build/$name/*.o -cudart static
echo build/$name.so
