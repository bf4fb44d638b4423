mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_dist.py -x -q -m gpu > gpurun_out/par.log 2>&1
echo parity rc=$? >> gpurun_out/par.log
for k in 1 2; do
for so in build/variants/*.so; do LMX_LIBRARY=$so timeout 300 python tools/variant_bench.py --steps 4; done
done > gpurun_out/var.log 2>&1
