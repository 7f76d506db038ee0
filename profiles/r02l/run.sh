# r02l: interim end-of-round capture -- full GPU suite (incl. C4/C5, sanitizers), smoke, full bench,
# reference arm, partitioned N=1, ncu launch list + --set full of the dominant kernels
set -x
python __graft_entry__.py build 2>&1 | tail -2
mkdir -p gpurun_out/r02l
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 --timeout-method thread --durations=15 2>&1 | tail -30 > gpurun_out/r02l/pytest_gpu.txt
tail -20 gpurun_out/r02l/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02l/smoke.txt 2>&1; tail -2 gpurun_out/r02l/smoke.txt
timeout 1500 python bench.py > gpurun_out/r02l/bench.json 2> gpurun_out/r02l/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/r02l/bench_reference.json 2>> gpurun_out/r02l/bench.err
timeout 900 python bench.py --partitioned --no-e2e --no-big --no-next > gpurun_out/r02l/bench_partitioned.json 2>> gpurun_out/r02l/bench.err
B="python bench.py --steps 1 --warmup 1 --no-next --no-e2e --no-cpu-baseline --no-big"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02l/launches.csv \
  $B > gpurun_out/r02l/launches_bench.log 2>&1
python profiles/summarize_launches.py gpurun_out/r02l/launches.csv gpurun_out/r02l/launches_summary.csv | head -30
for KS in k_spmv_sell:40 k_update:40 k_small_warp:3 k_num_large_atomic:1 k_tail:1 k_level0:1 k_tag:1 k_mid_warp:3; do
  K=${KS%%:*}; S=${KS##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 \
    -o gpurun_out/r02l/full_$K $B > gpurun_out/r02l/full_$K.log 2>&1
  ncu -i gpurun_out/r02l/full_$K.ncu-rep --page raw --csv > gpurun_out/r02l/full_${K}_raw.csv 2>/dev/null
done
python profiles/summarize_full.py gpurun_out/r02l > gpurun_out/r02l/summary.txt
cat gpurun_out/r02l/summary.txt | head -80
rm -f gpurun_out/r02l/*.ncu-rep
