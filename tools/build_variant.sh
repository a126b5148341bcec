#!/bin/bash
# Build an A/B variant of the library with extra -D flags:
#   tools/build_variant.sh <name> -DCL_HIST_U8=0 ...   -> build/variants/<name>.so
# then run with CHUNKLAB_LIB=build/variants/<name>.so.
set -e
cd "$(dirname "$0")/.."
name=$1; shift
out=build/variants/$name; rm -rf $out; mkdir -p $out
pids=()
for f in paper_2604_10597_b200/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC \
    --expt-relaxed-constexpr -Iinclude -Ipaper_2604_10597_b200/csrc "$@" -c $f -o $out/$(basename $f).o &
  pids+=($!)
done
for p in "${pids[@]}"; do wait $p; done  # any failed compile fails the build (set -e)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o build/variants/$name.so $out/*.o -lpthread -ldl -lrt
echo build/variants/$name.so
