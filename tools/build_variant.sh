#!/bin/bash
# Build the library with extra -D flags into paper_2512_20943_b200/lib/variants/NAME.so
# (A/B experiments; select at run time with AIRGS_B200_LIB=<path>).
#   tools/build_variant.sh NAME "-DCOMP_CHUNK=32 ..."
set -e
NAME=$1; DEFS=$2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=$ROOT/paper_2512_20943_b200/csrc
OUT=$ROOT/paper_2512_20943_b200/lib/variants/$NAME
mkdir -p $OUT
for f in api render codec delta metrics io; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -fmad=false \
    -Xcompiler -fPIC,-fvisibility=hidden --expt-relaxed-constexpr $DEFS -c $SRC/$f.cu -o $OUT/$f.o &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $OUT.so $OUT/*.o
echo $OUT.so
