set -x
python __graft_entry__.py build 2>&1 | tail -1
AGIPC_TAIL_TRACE=1 timeout 600 python profiles/r02p/trace_c3.py /tmp/t.txt 2>&1 | grep tail-trace | tail -4
