# r02k: 12-DoF chunks on a second stream next to the small / mid rows (symbolic and numeric)
set -x
python __graft_entry__.py build 2>&1 | tail -2
mkdir -p gpurun_out/r02k
export AGIPC_SKIP_FULL_CONFIGS=1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_comm_gpu.py tests/test_dist_gpu.py -q -x --timeout 600 --timeout-method thread 2>&1 | tail -3
for i in 1 2; do timeout 600 python bench.py --steps 10 --warmup 3 --no-next --no-e2e --no-cpu-baseline --no-big > gpurun_out/r02k/bench$i.json 2>> gpurun_out/r02k/bench.err; done
python - <<'PY'
import json
for i in (1, 2):
    d = json.load(open(f"gpurun_out/r02k/bench{i}.json"))
    print({k: d[k] for k in ("value", "ms_per_step", "pcg_iters_per_s")}, d["roofline"]["frac"], d["phase_ms_per_step"])
PY
