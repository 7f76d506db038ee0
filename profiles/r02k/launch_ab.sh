python __graft_entry__.py build 2>&1 | tail -1
for i in 1 2 3; do timeout 300 python profiles/r02f/probe.py c3 2>&1 | grep c3_coarsen; done
