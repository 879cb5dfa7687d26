#!/bin/bash
# Build an alternative libnif_b200.so with extra nvcc defines for one unit:
#   tools/build_variant.sh <tag> <unit.cu> <nvcc flags...>  -> variants/libnif_<tag>.so
# (select at run time with NIF_B200_LIB=variants/libnif_<tag>.so; variants/ travels to the GPU box)
set -e
mkdir -p "$(dirname "$0")/../variants"
cd "$(dirname "$0")/.."
tag=$1; unit=$2; shift 2
ARCH="-gencode arch=compute_100a,code=sm_100a"
COMMON="-O3 -std=c++17 -lineinfo -Xcompiler -fPIC,-ffp-contract=off --expt-relaxed-constexpr -I include -I paper_2306_07191_b200/csrc"
objs=""
for f in build/*.o; do
  b=$(basename $f .o)
  if [ "$b" == "$unit" ] || [[ "$b" == var_* ]]; then continue; fi
  objs="$objs $f"
done
mad=""
case $unit in trace.cu|exact.cu|gather.cu|train.cu) mad="-fmad=false";; esac
nvcc $ARCH $COMMON $mad "$@" -c paper_2306_07191_b200/csrc/$unit -o build/var_$tag.o
nvcc $ARCH -shared -cudart static -o variants/libnif_$tag.so $objs build/var_$tag.o -Xlinker --no-undefined -lpthread -ldl -lrt
echo variants/libnif_$tag.so
