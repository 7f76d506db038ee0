# r02v (12): register sort in k_group_unique, 32-entry symbolic list launched first, numeric
# 32-entry kernel skipped when the list is empty
set -x
python __graft_entry__.py build 2>&1 | tail -1
export AGIPC_SKIP_FULL_CONFIGS=1
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 --timeout-method thread 2>&1 | tail -3 > gpurun_out/parity.txt; cat gpurun_out/parity.txt
bash profiles/ab_libs.sh gpurun_out/r02v12 "base prev"
mkdir -p gpurun_out/r02v12
timeout 600 python profiles/r02p/trace_c3.py gpurun_out/r02v12/trace.txt 2>&1 | tail -1
python profiles/r02p/analyze_trace.py gpurun_out/r02v12/trace.txt k_tag | sed -n 17,40p
