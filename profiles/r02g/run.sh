# r02g: tail edges remapped in place (no compaction), L2 window only when the arena fits,
# flat K1 with 8-lane segments, factorised large kernel dropped
set -x
python __graft_entry__.py build 2>&1 | tail -2
mkdir -p gpurun_out/r02g
export AGIPC_SKIP_FULL_CONFIGS=1
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 --timeout-method thread --deselect tests/test_sanitizer_gpu.py 2>&1 | tail -4
timeout 300 python profiles/r02f/probe.py c3 > gpurun_out/r02g/probe_c3.jsonl 2> gpurun_out/r02g/probe.err
timeout 300 python profiles/r02f/probe.py c4 > gpurun_out/r02g/probe_c4.jsonl 2>> gpurun_out/r02g/probe.err
cat gpurun_out/r02g/probe_c3.jsonl gpurun_out/r02g/probe_c4.jsonl
timeout 1200 python bench.py --no-cpu-baseline > gpurun_out/r02g/bench.json 2> gpurun_out/r02g/bench.err
tail -2 gpurun_out/r02g/bench.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/r02g/bench.json"))
print({k: d[k] for k in ("value", "ms_per_step", "pcg_iters_per_s")}, d["roofline"]["frac"], d["phase_ms_per_step"])
print(json.dumps(d["single_gpu_configs"]))
print(json.dumps(d["next_rows"]))
print(json.dumps(d["e2e"]))
PY
