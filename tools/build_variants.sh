#!/bin/bash
# Build liblmx variants into build/variants/ for A/B timing on one box.
# usage: tools/build_variants.sh "NAME:FLAGS[:GITREV]" ...
#   FLAGS  extra -D macros for the round loops (lmx_round.cu, lmx_scan.cu)
#   GITREV take both round-loop sources from that git revision
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
CSRC=$ROOT/paper_1302_4587_b200/csrc
OBJ=$ROOT/build/obj
mkdir -p $ROOT/build/variants
rm -f $ROOT/build/variants/*.so
make -s -C $CSRC
for spec in "$@"; do
  name=$(echo "$spec" | cut -d: -f1); flags=$(echo "$spec" | cut -d: -f2); rev=$(echo "$spec" | cut -s -d: -f3)
  objs=""
  for f in lmx_round lmx_scan; do
    src=$CSRC/$f.cu
    if [ -n "$rev" ]; then
      src=/tmp/var_src_${name}_$f.cu
      git -C $ROOT show "$rev:paper_1302_4587_b200/csrc/$f.cu" > $src
    fi
    objs="$objs /tmp/var_${name}_$f.o"
    echo "$src" > /tmp/var_${name}_$f.src
  done
  ( for f in lmx_round lmx_scan; do
      nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC $flags -I$CSRC \
        -c $(cat /tmp/var_${name}_$f.src) -o /tmp/var_${name}_$f.o -Xptxas -v 2> /tmp/var_${name}_$f.ptxas || exit 1
    done &&
    nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $ROOT/build/variants/liblmx_$name.so \
      $objs $(ls $OBJ/*.o | grep -v -F -e /lmx_round.o -e /lmx_scan.o) -cudart static ) &
done
wait
ls $ROOT/build/variants
