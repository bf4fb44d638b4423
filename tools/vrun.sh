mkdir -p gpurun_out


for k in 1 2; do
for so in build/variants/*.so; do LMX_LIBRARY=$so timeout 300 python tools/variant_bench.py --steps 4; done
done > gpurun_out/var.log 2>&1
