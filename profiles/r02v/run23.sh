# r02v (23): k_clear_slots and k_apply folded into k_tail; host-time markers in the trace
set -x
python __graft_entry__.py build 2>&1 | tail -1
export AGIPC_SKIP_FULL_CONFIGS=1
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 --timeout-method thread 2>&1 | tail -2 > gpurun_out/parity.txt; cat gpurun_out/parity.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
bash profiles/ab_libs.sh gpurun_out/r02v23 "base prev"
mkdir -p gpurun_out/r02v23
timeout 600 python profiles/r02p/trace_c3.py gpurun_out/r02v23/trace.txt 2>&1 | tail -1
python profiles/r02p/analyze_trace.py gpurun_out/r02v23/trace.txt k_tag | head -14
