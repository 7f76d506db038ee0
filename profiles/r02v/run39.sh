set -x
python __graft_entry__.py build 2>&1 | tail -1
AGIPC_LIB=$PWD/variants/l0c1/libagipc.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "map or full" --timeout 600 --timeout-method thread 2>&1 | tail -1
bash profiles/ab_libs.sh gpurun_out/r02v39 "l0c2 l0c1"
