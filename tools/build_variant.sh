#!/bin/bash
# Build a variant of the library with extra nvcc defines (dev A/B of compile-time
# kernel options); load it with MIXTILE_LIB=<path>.
#   bash tools/build_variant.sh <name> -DMT_EPI_WARPS=8 ...
set -e
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
out=$root/paper_2003_05324_b200/_build/variants/$name
mkdir -p $out
objs=""
for u in api gen potrf trsm update solve prof tc_update tc2_update tc2w_update tcf_update dmma_update; do
  extra=""; [ $u = gen ] && extra="-fmad=false"
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    -I $root/include --expt-relaxed-constexpr $extra "$@" -c $root/paper_2003_05324_b200/csrc/$u.cu -o $out/$u.o &
  objs="$objs $out/$u.o"
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libmixtile_b200.so $objs -lpthread
echo $out/libmixtile_b200.so
