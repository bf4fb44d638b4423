mkdir -p gpurun_out
for k in 1 2; do
for so in build/variants/*.so; do LMX_LIBRARY=$so timeout 300 python tools/variant_bench.py --scale 24 --er --steps 4; done
done > gpurun_out/var_er.log 2>&1
