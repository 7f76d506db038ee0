python __graft_entry__.py build 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 --timeout-method thread -k "tag or full_size or shells or mixed" 2>&1 | tail -2
for i in 1 2; do timeout 300 python profiles/r02f/probe.py c3 2>&1 | grep c3_coarsen; done
