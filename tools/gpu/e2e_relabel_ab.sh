# A/B of the e2e leg's relabelling (RMAT-26): auto (on for skewed graphs) vs off
for i in 1 2; do
  for R in auto off; do
    timeout 400 python bench.py --no-cpu-baseline --steps 5 --warmup 3 --e2e-steps 4 --e2e-relabel $R > gpurun_out/b_e2e_${R}_$i.json 2> gpurun_out/b_e2e_${R}_$i.err
  done
done
