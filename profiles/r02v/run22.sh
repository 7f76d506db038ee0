# r02v (22): aux stream (large rows + mid nodes) at the highest stream priority vs default
set -x
python __graft_entry__.py build 2>&1 | tail -1
bash profiles/ab_libs.sh gpurun_out/r02v22 "base"
bash profiles/ab_libs.sh gpurun_out/r02v22o "base" AGIPC_AUX_PRIO=0
