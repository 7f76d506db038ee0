# r02c (2): interface records per chunk (list kept across batches), CTA-per-node reduction
set -x
python __graft_entry__.py build 2>&1 | tail -2
mkdir -p gpurun_out/r02c2
export AGIPC_SKIP_FULL_CONFIGS=1
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 --timeout-method thread --durations=10 \
   2>&1 | tail -30 > gpurun_out/r02c2/tests.txt
cat gpurun_out/r02c2/tests.txt
timeout 600 python bench.py --steps 10 --warmup 3 --no-next --no-e2e --no-cpu-baseline --no-big > gpurun_out/r02c2/bench.json 2> gpurun_out/r02c2/bench.err
tail -3 gpurun_out/r02c2/bench.err; head -c 2500 gpurun_out/r02c2/bench.json
B="python bench.py --steps 1 --warmup 1 --no-next --no-e2e --no-cpu-baseline --no-big"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02c2/launches.csv \
  $B > gpurun_out/r02c2/launches_bench.log 2>&1
python profiles/summarize_launches.py gpurun_out/r02c2/launches.csv gpurun_out/r02c2/launches_summary.csv | head -30
for KS in k_small_warp:2 k_num_large:1 k_large_reduce:1 k_tail:1 k_mid_warp:2; do
  K=${KS%%:*}; S=${KS##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 \
    -o gpurun_out/r02c2/full_$K $B > gpurun_out/r02c2/full_$K.log 2>&1
  ncu -i gpurun_out/r02c2/full_$K.ncu-rep --page raw --csv > gpurun_out/r02c2/full_${K}_raw.csv 2>/dev/null
done
ls -la gpurun_out/r02c2
