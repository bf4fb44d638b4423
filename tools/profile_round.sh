#!/bin/bash
# Round-end evidence on one B200: GPU tests, the bench line, the ncu launch
# list of one RMAT-26 matching, and ncu --set full captures of the scan-loop
# kernels.  Outputs land in gpurun_out/ (copy the ones to keep into profiles/).
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
python bench.py > gpurun_out/bench26.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --profile-from-start off --metrics $M --clock-control none --csv \
  --log-file gpurun_out/launches26.csv python tools/profile_step.py --scale 26 > gpurun_out/ncu_list.log 2>&1
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none \
  -k regex:"lmx_scan_round_kernel|lmx_scan_match_kernel" -c 5 -f -o gpurun_out/scan_kernels_rmat26 \
  python tools/profile_step.py --scale 26 > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none \
  -k regex:"lmx_scan_hist_hub_kernel|lmx_scan_edge_bits" -c 2 -f -o gpurun_out/hist_kernel_rmat26 \
  python tools/profile_step.py --scale 26 > gpurun_out/ncu_hist.log 2>&1
echo done
