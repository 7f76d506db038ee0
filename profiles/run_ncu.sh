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
# K:skip (launches to skip: the warm-up step's, or 40 PCG iterations)
for KS in k_spmv_sell:40 k_update:40 k_num_large:2 k_mid_warp:2 k_small_warp:4 k_tail:1 k_level0:1 k_tag:1 \
          k_cross_to_level1:1 k_sym_large:1; do
  K=${KS%%:*}; S=${KS##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 \
    -o $OUT/full_$K $B > $OUT/full_$K.log 2>&1
done
for f in $OUT/full_*.ncu-rep; do
  ncu -i $f --page raw --csv > ${f%.ncu-rep}_raw.csv 2>/dev/null
done
ls -la $OUT
