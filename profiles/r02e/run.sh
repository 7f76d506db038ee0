# r02e: absolute mirror positions, half-warp flat K1, k_level0 flush fence; full suite + full bench
set -x
python __graft_entry__.py build 2>&1 | tail -2
mkdir -p gpurun_out/r02e
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 --timeout-method thread --durations=12 \
   2>&1 | tail -60 > gpurun_out/r02e/tests.txt
grep -v "^E   " gpurun_out/r02e/tests.txt | tail -25
grep "^E   " gpurun_out/r02e/tests.txt | head -30
timeout 1200 python bench.py > gpurun_out/r02e/bench.json 2> gpurun_out/r02e/bench.err
tail -3 gpurun_out/r02e/bench.err; cat gpurun_out/r02e/bench.json
B="python bench.py --steps 1 --warmup 1 --no-next --no-e2e --no-cpu-baseline --no-big"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02e/launches.csv \
  $B > gpurun_out/r02e/launches_bench.log 2>&1
python profiles/summarize_launches.py gpurun_out/r02e/launches.csv gpurun_out/r02e/launches_summary.csv | head -30
