# r02z (check 2): full GPU suite + smoke + default bench after the level-0 tile change
set -x
python __graft_entry__.py build 2>&1 | tail -2
O=gpurun_out/r02z6
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 --timeout-method thread --durations=5 2>&1 | tail -10 > $O/pytest_gpu.txt
tail -2 $O/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
timeout 1500 python bench.py > $O/bench.json 2> $O/bench.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r02z6/bench.json").read().strip().splitlines()[-1])
p = d["phase_ms_per_step"]; b = d["single_gpu_configs"]
print(d["value"], d["ms_per_step"], d["pcg_iters_per_s"], d["roofline"]["frac"], d["e2e"]["value"], {k: p[k] for k in ("map_level0","map_tail","asm_classify","asm_symbolic","asm_numeric")}, b["C4"]["coarsen_assemble_ms"], b["C5"]["coarsen_assemble_ms"])
PY
