# late-round batching of the multi-GPU protocol (one rank over NCCL, RMAT-26): threshold x batch
echo "NCCL_DEBUG=${NCCL_DEBUG:-unset}" >> gpurun_out/late_sweep.txt
for cfg in ${LATE_CFGS:-"0 4" "4194304 4" "4194304 8" "16777216 4" "16777216 8" "67108864 8"}; do
  set -- $cfg
  LMX_DIST_LATE_FOUND=$1 LMX_DIST_LATE_BATCH=$2 timeout 300 python bench.py --dist --no-cpu-baseline --steps 10 --warmup 3 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('late_found $1 batch $2: %.3f ms per matching' % d['ms_per_step'])" >>> gpurun_out/late_sweep.txt
done
