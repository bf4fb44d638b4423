#!/bin/bash
# A/B the built variants (build/variants/*.so): ER-24 unit weights (compacting loop) and RMAT-24 (general
# layout forced? no: scan) -- 2 passes each, each run under its own timeout.
mkdir -p gpurun_out
for k in 1 2; do
for so in build/variants/*.so; do LMX_LIBRARY=$so timeout 120 python tools/variant_bench.py --scale 24 --er --steps 4; done
done > gpurun_out/var_er.log 2>&1
for k in 1 2; do
for so in build/variants/*.so; do LMX_LIBRARY=$so timeout 200 python tools/variant_bench.py --scale 24 --compact --steps 3; done
done > gpurun_out/var_rmat_compact.log 2>&1
