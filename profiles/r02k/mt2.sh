python __graft_entry__.py build 2>&1 | tail -1
AGIPC_TAIL_TRACE=1 timeout 300 python profiles/r02f/probe.py c3 2>&1 | grep -E "tail-trace|c3_coarsen" | tail -3
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_dist_gpu.py -q -x --timeout 300 --timeout-method thread -k "map or dist or full_size or c4" 2>&1 | tail -2
