python __graft_entry__.py build 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_dist_gpu.py -q -x --timeout 300 --timeout-method thread 2>&1 | tail -3
