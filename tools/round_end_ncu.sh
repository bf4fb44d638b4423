#!/bin/bash
# ncu evidence for the RMAT-26 matching (after the changed program ran clean):
#  1. launch list of 5 profiled matchings (time + DRAM bytes per launch, cold, serialised)
#  2. --set full capture of one lmx_scan_loop_kernel launch, and of the histogram kernel
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --profile-from-start off --metrics $M --clock-control none --csv \
  --log-file gpurun_out/launches26.csv python tools/profile_step.py --scale 26 --steps 5 > gpurun_out/ncu_list.log 2>&1
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none \
  -k regex:"lmx_scan_loop_kernel" -c 1 -f -o gpurun_out/loop_kernel_rmat26 \
  python tools/profile_step.py --scale 26 > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none \
  -k regex:"lmx_scan_hist_hub_kernel" -c 1 -f -o gpurun_out/hist_kernel_rmat26 \
  python tools/profile_step.py --scale 26 > gpurun_out/ncu_hist.log 2>&1
echo done
