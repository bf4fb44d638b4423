#!/bin/bash
# A/B the built variants (build/variants/*.so) on RMAT scale ${1:-26}, 2 passes.
mkdir -p gpurun_out
for k in 1 2; do
for so in build/variants/*.so; do LMX_LIBRARY=$so timeout 300 python tools/variant_bench.py --scale ${1:-26} --steps 4; done
done > gpurun_out/var_rmat.log 2>&1
