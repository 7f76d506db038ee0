# r02v (10): large rows from entry lists written by the symbolic pass (k_num_large_list) vs the
# classifying chunks (AGIPC_LARGE_LIST=0)
set -x
python __graft_entry__.py build 2>&1 | tail -1
export AGIPC_SKIP_FULL_CONFIGS=1
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 --timeout-method thread 2>&1 | tail -3 > gpurun_out/parity.txt; cat gpurun_out/parity.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
bash profiles/ab_libs.sh gpurun_out/r02v10 "base"
bash profiles/ab_libs.sh gpurun_out/r02v10o "base" AGIPC_LARGE_LIST=0
mkdir -p gpurun_out/r02v10
timeout 600 python profiles/r02p/trace_c3.py gpurun_out/r02v10/trace.txt 2>&1 | tail -2
python profiles/r02p/analyze_trace.py gpurun_out/r02v10/trace.txt k_tag | tail -14
