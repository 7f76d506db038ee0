# r02v (27): k_num_large_list occupancy -- 4 / 5 / 6 CTAs per SM (128 / 96 / 80 registers) with
# 96-entry interface batches (30 KB shared), vs the current 4 CTAs with 192-entry batches (base)
set -x
python __graft_entry__.py build 2>&1 | tail -1
bash profiles/ab_libs.sh gpurun_out/r02v27 "base m4s96 m5s96 m6s96"
