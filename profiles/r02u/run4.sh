set -x
python __graft_entry__.py build 2>&1 | tail -1
mkdir -p gpurun_out/r02u4
timeout 600 python profiles/r02p/trace_c3.py gpurun_out/r02u4/trace_c3.txt 2>&1 | tail -6
python profiles/r02p/analyze_trace.py gpurun_out/r02u4/trace_c3.txt k_tag
B="python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu-baseline --no-big"
timeout 600 $B > gpurun_out/r02u4/bench.json 2>> gpurun_out/r02u4/bench.err
python - gpurun_out/r02u4/bench.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
p = d["phase_ms_per_step"]; nx = d["next_rows"]["post_coarsening_pcg"]
print(f"value {d['value']:.4f} step {d['ms_per_step']:.3f} it/s {d['pcg_iters_per_s']} pcg_setup {p['pcg_setup']:.4f} next {nx['ms_per_solve']:.3f} next_phases {nx.get('phases_ms')}")
print(p)
PY
