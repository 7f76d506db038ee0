# r02p: launch trace of one warm C3 coarsen (AGIPC_TRACE): kernel durations vs idle gaps
set -x
python __graft_entry__.py build 2>&1 | tail -2
mkdir -p gpurun_out/r02p
timeout 600 python profiles/r02p/trace_c3.py gpurun_out/r02p/trace_c3.txt 2>&1 | tail -8
python profiles/r02p/analyze_trace.py gpurun_out/r02p/trace_c3.txt k_tag > gpurun_out/r02p/trace_summary.txt
cat gpurun_out/r02p/trace_summary.txt
