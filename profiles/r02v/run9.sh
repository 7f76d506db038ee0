# r02v (9): k_tail skips clean tiles (no intra-group edge at this level): no closure / rank pass,
# rank = offset in the tile
set -x
python __graft_entry__.py build 2>&1 | tail -1
export AGIPC_SKIP_FULL_CONFIGS=1
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 --timeout-method thread 2>&1 | tail -3 > gpurun_out/parity.txt; cat gpurun_out/parity.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
bash profiles/ab_libs.sh gpurun_out/r02v9 "base prev"
AGIPC_TAIL_TRACE=1 timeout 600 python profiles/r02p/trace_c3.py /tmp/t.txt 2>&1 | grep tail-trace | tail -3
