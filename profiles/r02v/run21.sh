# r02v (21): 12-DoF diagonal blocks factorised per fine row in k_num_large_list (base) vs per block (nofac)
set -x
python __graft_entry__.py build 2>&1 | tail -1
export AGIPC_SKIP_FULL_CONFIGS=1
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 --timeout-method thread 2>&1 | tail -2 > gpurun_out/parity.txt; cat gpurun_out/parity.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
bash profiles/ab_libs.sh gpurun_out/r02v21 "base nofac"
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-big --no-next"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_num_large_list --csv $B 2>/dev/null | grep k_num_large | tail -1 | awk -F, '{print "base large-list ns", $NF}'
