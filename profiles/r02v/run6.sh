# r02v (6): no host round trip after the classification (device-side list sizes); the one
# after the symbolic pass stays (sizes returned while the numeric pass runs asynchronously)
set -x
python __graft_entry__.py build 2>&1 | tail -1
export AGIPC_SKIP_FULL_CONFIGS=1
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 --timeout-method thread 2>&1 | tail -3 > gpurun_out/parity.txt; cat gpurun_out/parity.txt
bash profiles/ab_libs.sh gpurun_out/r02v6 "base prev"
