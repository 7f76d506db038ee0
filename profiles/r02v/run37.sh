# r02v (37): warp-aggregated pair count / scatter (base) vs HEAD (prev); scan tiles of 4096 / 1024 items
set -x
python __graft_entry__.py build 2>&1 | tail -1
export AGIPC_SKIP_FULL_CONFIGS=1
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 --timeout-method thread 2>&1 | tail -1
for n in scan16 scan4; do AGIPC_LIB=$PWD/variants/$n/libagipc.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 --timeout-method thread 2>&1 | tail -1; done
bash profiles/ab_libs.sh gpurun_out/r02v37 "base prev scan16 scan4"
