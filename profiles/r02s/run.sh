# r02s: source-level stall profiles of the large-row numeric chunks and the mid-node warps
set -x
python __graft_entry__.py build 2>&1 | tail -2
mkdir -p gpurun_out/r02s
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-big --no-next"
for KS in k_num_large_atomic:1 k_mid_warp:2 k_sym_large:1; do
  K=${KS%%:*}; S=${KS##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 \
    -o gpurun_out/r02s/full_$K $B > gpurun_out/r02s/full_$K.log 2>&1
  ncu -i gpurun_out/r02s/full_$K.ncu-rep --page raw --csv > gpurun_out/r02s/full_${K}_raw.csv 2>/dev/null
  ncu -i gpurun_out/r02s/full_$K.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r02s/src_$K.csv 2>/dev/null
  python profiles/stall_by_line.py gpurun_out/r02s/src_$K.csv > gpurun_out/r02s/stalls_$K.txt 2>&1
  head -30 gpurun_out/r02s/stalls_$K.txt
done
python profiles/summarize_full.py gpurun_out/r02s > gpurun_out/r02s/summary.txt; cat gpurun_out/r02s/summary.txt
rm -f gpurun_out/r02s/*.ncu-rep gpurun_out/r02s/src_*.csv
