#!/bin/bash
# Build liblmx variants into build/variants/ for A/B timing on one box.
# usage: tools/build_variants.sh "NAME:FLAGS[:GITREV]" ...
#   FLAGS  extra -D macros for lmx_round.cu
#   GITREV take lmx_round.cu from that git revision (A/B against older code)
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
CSRC=$ROOT/paper_1302_4587_b200/csrc
OBJ=$ROOT/build/obj
mkdir -p $ROOT/build/variants
rm -f $ROOT/build/variants/*.so
make -s -C $CSRC
for spec in "$@"; do
  name=$(echo "$spec" | cut -d: -f1); flags=$(echo "$spec" | cut -d: -f2); rev=$(echo "$spec" | cut -s -d: -f3)
  src=$CSRC/lmx_round.cu
  if [ -n "$rev" ]; then
    src=/tmp/var_src_$name.cu
    git -C $ROOT show "$rev:paper_1302_4587_b200/csrc/lmx_round.cu" > $src
  fi
  ( nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC $flags -I$CSRC \
      -c $src -o /tmp/var_$name.o -Xptxas -v 2> /tmp/var_$name.ptxas &&
    nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $ROOT/build/variants/liblmx_$name.so \
      /tmp/var_$name.o $OBJ/lmx_setup.o $OBJ/lmx_capi.o $OBJ/lmx_build.o $OBJ/lmx_coarsen.o -cudart static ) &
done
wait
ls $ROOT/build/variants
