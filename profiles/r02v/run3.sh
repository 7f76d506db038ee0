# r02v (3): k_tail grid barrier -- release/acquire (base) vs fences + nanosleep (bar0) vs cg grid.sync
set -x
python __graft_entry__.py build 2>&1 | tail -1
export AGIPC_SKIP_FULL_CONFIGS=1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 --timeout-method thread -k "map or level or tail or full" 2>&1 | tail -2 > gpurun_out/parity.txt; cat gpurun_out/parity.txt
bash profiles/ab_libs.sh gpurun_out/r02v3 "base bar0"
bash profiles/ab_libs.sh gpurun_out/r02v3c "base" AGIPC_TAIL_COOP=1
