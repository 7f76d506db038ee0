# r02v (14): host waits spin on an event (no blocking-sync wake-up) at the map / assemble / PCG
# status sync points
set -x
python __graft_entry__.py build 2>&1 | tail -1
export AGIPC_SKIP_FULL_CONFIGS=1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_comm_gpu.py -q -x --timeout 600 --timeout-method thread 2>&1 | tail -2 > gpurun_out/parity.txt; cat gpurun_out/parity.txt
bash profiles/ab_libs.sh gpurun_out/r02v14 "base prev"
for n in base prev; do python - gpurun_out/r02v14/bench_$n.json $n <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[2], "step", d["ms_per_step"], "pcg it/s", d["pcg_iters_per_s"])
PY
done
