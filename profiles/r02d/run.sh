# r02d: deterministic child order, flat K1 for short solves, per-slice pq reduction, sanitizers
set -x
python __graft_entry__.py build 2>&1 | tail -2
mkdir -p gpurun_out/r02d
export AGIPC_SKIP_FULL_CONFIGS=1
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 --timeout-method thread --durations=12 \
   2>&1 | tail -60 > gpurun_out/r02d/tests.txt
grep -v "^E   " gpurun_out/r02d/tests.txt | tail -30
grep "^E   " gpurun_out/r02d/tests.txt | head -30
timeout 900 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-big > gpurun_out/r02d/bench.json 2> gpurun_out/r02d/bench.err
tail -3 gpurun_out/r02d/bench.err; head -c 3500 gpurun_out/r02d/bench.json
B="python bench.py --steps 1 --warmup 1 --no-next --no-e2e --no-cpu-baseline --no-big"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_small_warp -s 3 -c 1 \
    -o gpurun_out/r02d/full_k_small_warp $B > gpurun_out/r02d/full_k_small_warp.log 2>&1
ncu -i gpurun_out/r02d/full_k_small_warp.ncu-rep --page raw --csv > gpurun_out/r02d/full_k_small_warp_raw.csv 2>/dev/null
ncu -i gpurun_out/r02d/full_k_small_warp.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r02d/src_k_small_warp.csv 2>/dev/null
python profiles/stall_by_line.py gpurun_out/r02d/src_k_small_warp.csv 30
