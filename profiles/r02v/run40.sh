# r02v (40): k_num_large_list grid: 4 / 8 / 16 CTAs per SM (persistent, the next-chunk prefetch in use) vs 64
set -x
python __graft_entry__.py build 2>&1 | tail -1
bash profiles/ab_libs.sh gpurun_out/r02v40 "base lg4 lg8 lg16"
