# r02u (3): thread-per-row k_init (PCG setup of the coarse and the fine static solve)
set -x
python __graft_entry__.py build 2>&1 | tail -1
export AGIPC_SKIP_FULL_CONFIGS=1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_comm_gpu.py tests/test_dist_gpu.py -q -x --timeout 600 --timeout-method thread 2>&1 | tail -3
timeout 600 python profiles/r02u/trace_fine.py gpurun_out/r02u/trace_fine2.txt 2>&1 | tail -4
python profiles/r02p/analyze_trace.py gpurun_out/r02u/trace_fine2.txt k_dinv | tail -8
B="python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu-baseline --no-big"
timeout 600 $B > gpurun_out/r02u/bench3.json 2>> gpurun_out/r02u/bench.err
python - gpurun_out/r02u/bench3.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
p = d["phase_ms_per_step"]; nx = d["next_rows"]["post_coarsening_pcg"]
print(f"value {d['value']:.4f} step {d['ms_per_step']:.3f} it/s {d['pcg_iters_per_s']} pcg_setup {p['pcg_setup']:.4f} next {nx['ms_per_solve']:.3f} next_phases {nx.get('phases_ms')}")
PY
