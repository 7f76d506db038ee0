# r02v (16): timing experiment -- k_level0 without its decoupled look-back (wrong map, timing only)
set -x
python __graft_entry__.py build 2>&1 | tail -1
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-big --no-next"
mkdir -p gpurun_out/r02v16
for n in base nolb; do
  if [ "$n" = base ]; then L=""; else L="AGIPC_LIB=$PWD/variants/$n/libagipc.so"; fi
  env $L timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_level0 --csv $B 2>/dev/null | grep k_level0 | tail -2
done
