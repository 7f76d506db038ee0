python __graft_entry__.py build 2>&1 | tail -1
mkdir -p gpurun_out/r02k
for M in 4 5 4 5; do AGIPC_SMALL_MINB=$M timeout 300 python profiles/r02f/probe.py c3 2>/dev/null | head -1; done
