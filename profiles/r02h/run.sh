# r02h: L2 carve-out only while a fitting window is in use; all-cores oracle baseline; full bench
set -x
python __graft_entry__.py build 2>&1 | tail -2
mkdir -p gpurun_out/r02h
export AGIPC_SKIP_FULL_CONFIGS=1
timeout 900 python -m pytest tests -m gpu -q --timeout 600 --timeout-method thread --deselect tests/test_sanitizer_gpu.py 2>&1 | tail -4
timeout 300 python profiles/r02f/probe.py c4 > gpurun_out/r02h/probe_c4.jsonl 2> gpurun_out/r02h/probe.err
cat gpurun_out/r02h/probe_c4.jsonl
timeout 1500 python bench.py > gpurun_out/r02h/bench.json 2> gpurun_out/r02h/bench.err
tail -2 gpurun_out/r02h/bench.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/r02h/bench.json"))
print({k: d[k] for k in ("value", "ms_per_step", "pcg_iters_per_s")}, d["roofline"]["frac"], d["phase_ms_per_step"])
print(json.dumps(d["single_gpu_configs"]))
print(json.dumps(d["next_rows"]))
print(json.dumps(d["e2e"]))
print(json.dumps(d["cpu_baseline"]))
PY
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02h/bench_ref.json 2>> gpurun_out/r02h/bench.err
cat gpurun_out/r02h/bench_ref.json
