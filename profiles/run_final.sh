#!/bin/bash
# end-of-round capture: smoke, every GPU test, bench lines (default, reference arm, symmetric
# solve, partitioned path at N=1 over NCCL), launch list, ncu --set full of the top kernels
OUT=gpurun_out/${TAG:-final}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo smoke=$? >> $OUT/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo rc=$? >> $OUT/pytest_gpu.log
timeout 600 python bench.py > $OUT/bench.jsonl 2> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_reference.jsonl 2> $OUT/bench_reference.err
timeout 600 python bench.py --partitioned --no-cpu-baseline --no-next > $OUT/bench_partitioned.jsonl 2> $OUT/bench_partitioned.err
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $B > $OUT/launches_bench.log 2>&1
for KS in k_spmv_sell:40 k_update:40 k_num_large:1 k_small_warp:3; do
  K=${KS%%:*}; S=${KS##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 -o $OUT/full_$K $B > $OUT/full_$K.log 2>&1
  ncu -i $OUT/full_$K.ncu-rep --page raw --csv > $OUT/full_${K}_raw.csv 2>/dev/null
done
ls -la $OUT
