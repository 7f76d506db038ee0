#!/bin/bash
# ncu captures for profiles/ (run under gpurun on one B200).  Usage: bash profiles/run_ncu.sh TAG
set -x
TAG=${1:-r01}
OUT=gpurun_out/ncu_$TAG
mkdir -p $OUT
# 1) every launch of one warm step with its device time (cold-cache, serialised)
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/launches_bench.log 2>&1
# 2) full sets of the top kernels
for K in k_spmv_pq k_num_large k_num_small k_group_pass k_tag k_update; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 8 -c 2 \
    -o $OUT/full_$K python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/full_$K.log 2>&1
done
ls -la $OUT
