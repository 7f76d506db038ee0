# r02s (2): large-row chunks -- interface blocks staged 32 at a time, diagonal position and first
# 12-DoF column precomputed (no per-chunk binary searches)
set -x
python __graft_entry__.py build 2>&1 | tail -2
mkdir -p gpurun_out/r02s
export AGIPC_SKIP_FULL_CONFIGS=1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 --timeout-method thread 2>&1 | tail -4
B="python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-big --no-next"
for rep in 1 2; do
  timeout 600 $B > gpurun_out/r02s/bench$rep.json 2>> gpurun_out/r02s/bench.err
  python - $rep <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/r02s/bench{sys.argv[1]}.json").read().strip().splitlines()[-1])
p = d["phase_ms_per_step"]
print("rep", sys.argv[1], d["value"], d["pcg_iters_per_s"], {k: p[k] for k in ("asm_classify", "asm_symbolic", "asm_numeric", "map_tail")})
PY
done
K=k_num_large_atomic
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 -o gpurun_out/r02s/full2_$K $B --steps 1 --warmup 1 > /dev/null 2>&1
ncu -i gpurun_out/r02s/full2_$K.ncu-rep --page raw --csv > gpurun_out/r02s/full2_${K}_raw.csv 2>/dev/null
ncu -i gpurun_out/r02s/full2_$K.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r02s/src2_$K.csv 2>/dev/null
python profiles/stall_by_line.py gpurun_out/r02s/src2_$K.csv > gpurun_out/r02s/stalls2_$K.txt 2>&1
head -24 gpurun_out/r02s/stalls2_$K.txt
mkdir -p gpurun_out/r02s2; mv gpurun_out/r02s/full2_${K}_raw.csv gpurun_out/r02s2/
python profiles/summarize_full.py gpurun_out/r02s2 | head -20
rm -f gpurun_out/r02s/*.ncu-rep gpurun_out/r02s/src*.csv
