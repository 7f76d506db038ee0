# r02v (13): 32-bit symbolic sort keys (n_c < 2^26), numeric small rows read their children as
# the symbolic pass left them (no child_ptr -> child_list chain in the prefetch)
set -x
python __graft_entry__.py build 2>&1 | tail -1
export AGIPC_SKIP_FULL_CONFIGS=1
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 --timeout-method thread 2>&1 | tail -3 > gpurun_out/parity.txt; cat gpurun_out/parity.txt
bash profiles/ab_libs.sh gpurun_out/r02v13 "base prev"
