# r02v (33): k_large_rows_init on the aux stream (before the 12-DoF chunks) instead of before the fork
set -x
python __graft_entry__.py build 2>&1 | tail -1
export AGIPC_SKIP_FULL_CONFIGS=1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_skew.py -q -x --timeout 600 --timeout-method thread 2>&1 | tail -1
bash profiles/ab_libs.sh gpurun_out/r02v33 "base prev"
