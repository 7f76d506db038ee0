# r02v (11): numeric schedule A/B with the list-driven large rows (AGIPC_NUM_MODE 0 = aux stream
# overlap, 1 = large first then small on one stream, 2 = small first)
set -x
python __graft_entry__.py build 2>&1 | tail -1
bash profiles/ab_libs.sh gpurun_out/r02v11m0 "base"
bash profiles/ab_libs.sh gpurun_out/r02v11m1 "base" AGIPC_NUM_MODE=1
bash profiles/ab_libs.sh gpurun_out/r02v11m2 "base" AGIPC_NUM_MODE=2
