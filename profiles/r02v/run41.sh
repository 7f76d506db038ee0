# r02v (41): grid sizes of the small-row kernels (6 / 12 vs 32 CTAs per SM) and of k_sym_large (16 / 32 vs 64)
set -x
python __graft_entry__.py build 2>&1 | tail -1
export AGIPC_SKIP_FULL_CONFIGS=1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 --timeout-method thread 2>&1 | tail -1
bash profiles/ab_libs.sh gpurun_out/r02v41 "base sg6 sg12 slg16 slg32"
