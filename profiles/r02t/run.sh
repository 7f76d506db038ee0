# r02t: CTA-per-node mid kernels (k_mid_cta) vs warp-per-node (AGIPC_MID_WARP=1)
set -x
python __graft_entry__.py build 2>&1 | tail -1
export AGIPC_SKIP_FULL_CONFIGS=1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 --timeout-method thread 2>&1 | tail -4
bash profiles/ab_libs.sh gpurun_out/r02t "base"
bash profiles/ab_libs.sh gpurun_out/r02t_old "base" AGIPC_MID_WARP=1
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-big --no-next"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02t/launches.csv $B > /dev/null 2>&1
python profiles/summarize_launches.py gpurun_out/r02t/launches.csv gpurun_out/r02t/launches_summary.csv | head -30
