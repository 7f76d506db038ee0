# r02o: A x0 fused into the SELL value fill (post-coarsening fine solve), determinism-safe refine
# test, bench big configs with 2 warm-up steps; ncu of the small-row kernels
set -x
python __graft_entry__.py build 2>&1 | tail -2
mkdir -p gpurun_out/r02o
export AGIPC_SKIP_FULL_CONFIGS=1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_comm_gpu.py tests/test_dist_gpu.py tests/test_gpu_symmetric.py -q -x --timeout 600 --timeout-method thread 2>&1 | tail -5
for i in 1 2; do
  timeout 900 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-big > gpurun_out/r02o/bench$i.json 2>> gpurun_out/r02o/bench.err
done
python - <<'PY'
import json
for i in (1, 2):
    try:
        d = json.loads(open(f"gpurun_out/r02o/bench{i}.json").read().strip().splitlines()[-1])
    except Exception as e:
        print("bench", i, "failed", e); continue
    print({k: d.get(k) for k in ("value", "ms_per_step", "pcg_iters_per_s")}, d["roofline"]["frac"], d.get("phase_ms_per_step"))
    print("next:", d.get("next_rows", {}).get("post_coarsening_pcg"))
PY
B="python bench.py --steps 1 --warmup 1 --no-next --no-e2e --no-cpu-baseline --no-big"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02o/launches.csv $B > /dev/null 2>&1
python profiles/summarize_launches.py gpurun_out/r02o/launches.csv gpurun_out/r02o/launches_summary.csv | head -24
