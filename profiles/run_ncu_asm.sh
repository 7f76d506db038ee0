#!/bin/bash
# ncu --set full of the assembly numeric kernels (one launch each, the timed step's)
TAG=${1:-r01}
OUT=gpurun_out/ncu_$TAG
mkdir -p $OUT
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
for KS in "k_num_large:1" "k_mid_warp:3" "k_small_warp:3" "k_level0:1"; do
  K=${KS%%:*}; S=${KS##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 \
    -o $OUT/full_$K $B > $OUT/full_$K.log 2>&1
  ncu -i $OUT/full_$K.ncu-rep --page raw --csv > $OUT/full_${K}_raw.csv 2>/dev/null
done
ls -la $OUT
