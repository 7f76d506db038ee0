#!/bin/bash
# ncu --set full of the coarsen+assemble kernels of one timed C3 step (one launch each)
OUT=gpurun_out/ncu_r01i
mkdir -p $OUT
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-next"
for KS in "k_tail:1" "k_small_warp:3" "k_num_large:1" "k_mid_warp:3" "k_level0:1" "k_sym_small|k_group_unique:1"; do
  K=${KS%%:*}; S=${KS##*:}; N=$(echo $K | tr '|' '_')
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$K" -s $S -c 1 \
    -o $OUT/full_$N $B > $OUT/full_$N.log 2>&1
  ncu -i $OUT/full_$N.ncu-rep --page raw --csv > $OUT/full_${N}_raw.csv 2>/dev/null
  ncu -i $OUT/full_$N.ncu-rep --page source --csv > $OUT/full_${N}_source.csv 2>/dev/null
done
ls -la $OUT
