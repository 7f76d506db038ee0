#!/bin/bash
# ncu captures for profiles/ (run under gpurun on one B200).  Usage: bash profiles/run_ncu.sh TAG
# 1) the launch list of one warm step (gpu__time_duration per launch; cold-cache, serialised)
# 2) `--set full` of the top kernels (one or two launches each) -> dram bytes, stalls, source
set -x
TAG=${1:-r01}
OUT=gpurun_out/ncu_$TAG
mkdir -p $OUT
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  $B > $OUT/launches_bench.log 2>&1
for K in k_spmv_sell k_num_large k_mid_warp k_small_warp k_tail k_level0 k_update k_tag; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 40 -c 1 \
    -o $OUT/full_$K $B > $OUT/full_$K.log 2>&1
done
for f in $OUT/full_*.ncu-rep; do
  ncu -i $f --page raw --csv > ${f%.ncu-rep}_raw.csv 2>/dev/null
done
ls -la $OUT
