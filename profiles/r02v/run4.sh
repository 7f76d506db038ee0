# r02v (4): warp-cooperative staging of the scattered 72-B fine blocks (small-row parking,
# large-row diagonal and interface staging) vs lane-per-block loads (coop0)
set -x
python __graft_entry__.py build 2>&1 | tail -1
export AGIPC_SKIP_FULL_CONFIGS=1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 --timeout-method thread 2>&1 | tail -2 > gpurun_out/parity.txt; cat gpurun_out/parity.txt
bash profiles/ab_libs.sh gpurun_out/r02v4 "base coop0"
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-big --no-next"
mkdir -p gpurun_out/r02v4n
for KS in k_num_large_atomic:1 k_small_warp:3; do
  K=${KS%%:*}; S=${KS##*:}
  timeout 600 ncu --set full --clock-control none -k regex:$K -s $S -c 1 -o gpurun_out/r02v4n/full_$K $B > /dev/null 2>&1
  ncu -i gpurun_out/r02v4n/full_$K.ncu-rep --page raw --csv > gpurun_out/r02v4n/full_${K}_raw.csv 2>/dev/null
done
python profiles/summarize_full.py gpurun_out/r02v4n
rm -f gpurun_out/r02v4n/*.ncu-rep
