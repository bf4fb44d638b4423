for V in 0 2 1; do LMX_HIST_V2=$V timeout 400 python bench.py --no-cpu-baseline --no-e2e --steps 10 --warmup 3 > gpurun_out/b_h$V.json 2> gpurun_out/b_h$V.err; done
timeout 900 python -m pytest tests/test_dist.py tests/test_gpu_parity.py tests/test_gpu_scale.py -x -q -m gpu > gpurun_out/t_2p.log 2>&1
timeout 600 python bench.py --dist --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/b_dist1.json 2> gpurun_out/b_dist1.err
timeout 900 python bench.py --workload rmat27 --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/b_rmat27g.json 2> gpurun_out/b_rmat27g.err
