# r02v (34): k_task_node + k_fine_class + k_small_lists fused into k_class_lists
set -x
python __graft_entry__.py build 2>&1 | tail -1
export AGIPC_SKIP_FULL_CONFIGS=1
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 --timeout-method thread 2>&1 | tail -1
bash profiles/ab_libs.sh gpurun_out/r02v34 "base prev"
