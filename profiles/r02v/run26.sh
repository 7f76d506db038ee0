# r02v (26): symbolic tail fused (k_sym_finish = scalars + row pointer copy + mirror positions;
# pair scatter without the cursor copy)
set -x
python __graft_entry__.py build 2>&1 | tail -1
export AGIPC_SKIP_FULL_CONFIGS=1
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 --timeout-method thread 2>&1 | tail -2 > gpurun_out/parity.txt; cat gpurun_out/parity.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
bash profiles/ab_libs.sh gpurun_out/r02v26 "base prev"
