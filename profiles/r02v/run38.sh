# r02v (38): k_level0 chunks per warp (2 / 8 vs 4), k_cross_to_level1 grid (32 vs 8 CTAs per SM)
set -x
python __graft_entry__.py build 2>&1 | tail -1
for n in l0c2 l0c8 cg32; do AGIPC_LIB=$PWD/variants/$n/libagipc.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "map or full" --timeout 600 --timeout-method thread 2>&1 | tail -1; done
bash profiles/ab_libs.sh gpurun_out/r02v38 "base l0c2 l0c8 cg32"
