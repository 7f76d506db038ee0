# r02t (2): register-resident bitonic sort of the mid-node keys (k_mid_warp<false>)
set -x
python __graft_entry__.py build 2>&1 | tail -1
export AGIPC_SKIP_FULL_CONFIGS=1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 --timeout-method thread 2>&1 | tail -4
bash profiles/ab_libs.sh gpurun_out/r02t2 "base"
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-big --no-next"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02t2/launches.csv $B > /dev/null 2>&1
python profiles/summarize_launches.py gpurun_out/r02t2/launches.csv gpurun_out/r02t2/launches_summary.csv | sed -n 3,16p
