# r02v (42): grid of the mid-node kernels (4 / 6 / 24 vs 12 CTAs per SM)
set -x
python __graft_entry__.py build 2>&1 | tail -1
bash profiles/ab_libs.sh gpurun_out/r02v42 "base mg4 mg6 mg24"
