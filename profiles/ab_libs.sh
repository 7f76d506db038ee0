#!/bin/bash
# A/B of library variants on C3: bash profiles/ab_libs.sh OUTDIR "name1 name2 ..." [extra env, e.g. AGIPC_NUM_MODE=1]
# ("base" = the in-tree build; other names = variants/NAME/libagipc.so from profiles/build_variant.sh)
OUT=$1; NAMES=$2; EXTRA=$3
mkdir -p $OUT
B="python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-big --no-next"
for rep in 1 2; do
for n in $NAMES; do
  if [ "$n" = base ]; then L=""; else L="AGIPC_LIB=$PWD/variants/$n/libagipc.so"; fi
  env $L $EXTRA timeout 600 $B > $OUT/bench_$n.json 2>> $OUT/bench.err
  python - $OUT/bench_$n.json $n <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
except Exception as e:
    print(sys.argv[2], "FAILED", e); sys.exit(0)
p = d["phase_ms_per_step"]
print(f"{sys.argv[2]:10s} value {d['value']:.4f} it/s {d['pcg_iters_per_s']:.0f}", {k: p[k] for k in ("tag_edges", "map_level0", "map_tail", "asm_classify", "asm_symbolic", "asm_numeric")})
PY
done
done
