# r02u: software-pipelined SELL value fill (two blocks in flight per lane) vs the previous loop
set -x
python __graft_entry__.py build 2>&1 | tail -1
mkdir -p gpurun_out/r02u
export AGIPC_SKIP_FULL_CONFIGS=1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 --timeout-method thread -k "pcg or refine or prolong or static" 2>&1 | tail -3
B="python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu-baseline --no-big"
for rep in 1 2; do for n in base fill0; do
  if [ "$n" = base ]; then L=""; else L="AGIPC_LIB=$PWD/variants/$n/libagipc.so"; fi
  env $L timeout 600 $B > gpurun_out/r02u/bench_$n.json 2>> gpurun_out/r02u/bench.err
  python - gpurun_out/r02u/bench_$n.json $n <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
p = d["phase_ms_per_step"]; nx = d["next_rows"]["post_coarsening_pcg"]
print(f"{sys.argv[2]:6s} value {d['value']:.4f} step {d['ms_per_step']:.3f} pcg_setup {p['pcg_setup']:.4f} next {nx['ms_per_solve']:.3f} next_phases {nx.get('phases_ms')}")
PY
done; done
K=k_sell_fill
timeout 600 ncu --set full --clock-control none -k regex:$K -s 1 -c 1 -o gpurun_out/r02u/full_$K $B --steps 1 --warmup 1 --no-next > /dev/null 2>&1
ncu -i gpurun_out/r02u/full_$K.ncu-rep --page raw --csv > gpurun_out/r02u/full_${K}_raw.csv 2>/dev/null
python profiles/summarize_full.py gpurun_out/r02u
rm -f gpurun_out/r02u/*.ncu-rep
