# r02r: output-parallel numeric pass of the small coarse rows (k_small_warp<SEG, true>)
set -x
python __graft_entry__.py build 2>&1 | tail -2
mkdir -p gpurun_out/r02r
export AGIPC_SKIP_FULL_CONFIGS=1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 --timeout-method thread 2>&1 | tail -4
B="python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-big --no-next"
for rep in 1 2; do
  timeout 600 $B > gpurun_out/r02r/bench$rep.json 2>> gpurun_out/r02r/bench.err
  python - $rep <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/r02r/bench{sys.argv[1]}.json").read().strip().splitlines()[-1])
p = d["phase_ms_per_step"]
print("rep", sys.argv[1], d["value"], d["pcg_iters_per_s"], {k: p[k] for k in ("asm_classify", "asm_symbolic", "asm_numeric", "map_tail")})
PY
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_small_warp -s 3 -c 1 -o gpurun_out/r02r/full_small $B --steps 1 --warmup 1 > /dev/null 2>&1
ncu -i gpurun_out/r02r/full_small.ncu-rep --page raw --csv > gpurun_out/r02r/full_small_raw.csv 2>/dev/null
python profiles/summarize_full.py gpurun_out/r02r | head -20
rm -f gpurun_out/r02r/*.ncu-rep
