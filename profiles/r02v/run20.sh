set -x
python __graft_entry__.py build 2>&1 | tail -1
mkdir -p gpurun_out/r02v20
timeout 600 python profiles/r02p/trace_c3.py gpurun_out/r02v20/trace.txt 2>&1 | tail -2
python profiles/r02p/analyze_trace.py gpurun_out/r02v20/trace.txt k_tag
