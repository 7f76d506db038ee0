# r02q: A/B of the numeric-phase schedule (AGIPC_NUM_MODE 0 = 12-DoF chunks on the aux stream
# next to the small rows, 1 = chunks first on one stream, 2 = small rows first on one stream)
set -x
python __graft_entry__.py build 2>&1 | tail -2
mkdir -p gpurun_out/r02q
B="python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-big --no-next"
for rep in 1 2; do
for M in 0 1 2; do
  AGIPC_NUM_MODE=$M timeout 600 $B > gpurun_out/r02q/bench_m$M.json 2>> gpurun_out/r02q/bench.err
  python - $M <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/r02q/bench_m{sys.argv[1]}.json").read().strip().splitlines()[-1])
p = d["phase_ms_per_step"]
print("mode", sys.argv[1], d["value"], {k: p[k] for k in ("asm_classify", "asm_symbolic", "asm_numeric", "map_tail")})
PY
done
done
