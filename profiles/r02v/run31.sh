# r02v (31): k_tail tile size (TAIL_SUB 1 / 4) and 512-thread CTAs
set -x
python __graft_entry__.py build 2>&1 | tail -1
export AGIPC_SKIP_FULL_CONFIGS=1
for n in ts1 ts4 tt512; do AGIPC_LIB=$PWD/variants/$n/libagipc.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "map or full" --timeout 600 --timeout-method thread 2>&1 | tail -1; done
bash profiles/ab_libs.sh gpurun_out/r02v31 "base ts1 ts4 tt512"
