# r02v (2): 64 diagonal blocks staged per round (2 loads per lane) with 128-entry batches
set -x
python __graft_entry__.py build 2>&1 | tail -1
export AGIPC_SKIP_FULL_CONFIGS=1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 --timeout-method thread 2>&1 | tail -3 > gpurun_out/parity.txt; cat gpurun_out/parity.txt
bash profiles/ab_libs.sh gpurun_out/r02v2 "base d32 d32s128"
