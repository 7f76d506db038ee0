# r02v (25): k_tag occupancy variants (launch bounds min blocks 3 / 5 vs default)
set -x
python __graft_entry__.py build 2>&1 | tail -1
bash profiles/ab_libs.sh gpurun_out/r02v25 "base tag5 tag3"
