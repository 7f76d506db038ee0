python __graft_entry__.py build 2>&1 | tail -1
AGIPC_TAIL_TRACE=1 timeout 300 python profiles/r02f/probe.py c3 2>&1 | grep -E "tail-trace|c3_coarsen" | tail -6
