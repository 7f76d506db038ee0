set -x
python __graft_entry__.py build 2>&1 | tail -1
mkdir -p gpurun_out/r02u
timeout 600 python profiles/r02u/trace_fine.py gpurun_out/r02u/trace_fine.txt 2>&1 | tail -5
python profiles/r02p/analyze_trace.py gpurun_out/r02u/trace_fine.txt k_dinv | tail -40
