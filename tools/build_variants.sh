#!/bin/bash
# Build liblmx variants with different -D tuning macros into build/variants/.
# usage: tools/build_variants.sh "NAME:-DLMX_PAIRS=2 -DLMX_MINB=8" ...
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
CSRC=$ROOT/paper_1302_4587_b200/csrc
OBJ=$ROOT/build/obj
mkdir -p $ROOT/build/variants
rm -f $ROOT/build/variants/*.so
make -s -C $CSRC
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  ( nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC $flags \
      -c $CSRC/lmx_round.cu -o /tmp/var_$name.o -Xptxas -v 2> /tmp/var_$name.ptxas &&
    nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $ROOT/build/variants/liblmx_$name.so \
      /tmp/var_$name.o $OBJ/lmx_setup.o $OBJ/lmx_capi.o $OBJ/lmx_build.o -cudart static ) &
done
wait
ls $ROOT/build/variants
