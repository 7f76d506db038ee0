set -x
python __graft_entry__.py build 2>&1 | tail -1
mkdir -p gpurun_out/r02v8
AGIPC_NUM_MODE=1 timeout 600 python profiles/r02p/trace_c3.py gpurun_out/r02v8/trace_serial.txt 2>&1 | tail -3
python profiles/r02p/analyze_trace.py gpurun_out/r02v8/trace_serial.txt k_tag | tail -12
timeout 600 python profiles/r02p/trace_c3.py gpurun_out/r02v8/trace_conc.txt 2>&1 | tail -3
python profiles/r02p/analyze_trace.py gpurun_out/r02v8/trace_conc.txt k_tag
