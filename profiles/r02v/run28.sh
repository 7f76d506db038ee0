# r02v (28): occupancy of the symbolic mid-node warps (6 / 8 CTAs of 4 warps per SM: 80 / 64 regs)
# and of the symbolic small rows (6 CTAs of 8 warps: 40 regs) vs the plain bounds
set -x
python __graft_entry__.py build 2>&1 | tail -1
bash profiles/ab_libs.sh gpurun_out/r02v28 "base mids6 mids8 smalls6"
