mkdir -p gpurun_out
python -m pytest tests -x -q -m gpu > gpurun_out/par.log 2>&1
echo parity rc=$? >> gpurun_out/par.log
python bench.py > gpurun_out/bench_spec.log 2>&1
python tools/configs.py > gpurun_out/configs.log 2>&1
