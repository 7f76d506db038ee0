# r02v: large-row chunks -- two-stage phase-1 pipeline, diagonal accumulator flushed per batch
set -x
python __graft_entry__.py build 2>&1 | tail -1
export AGIPC_SKIP_FULL_CONFIGS=1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 --timeout-method thread 2>&1 | tail -3
bash profiles/ab_libs.sh gpurun_out/r02v "base prev"
