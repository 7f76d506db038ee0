# r02z: end-of-round capture at the final code -- full GPU suite (C4 / C5 full size), smoke, full
# bench, reference arm, partitioned path at N=1, C5 strong-scaling line at N=1, launch trace of a
# warm C3 coarsen, ncu launch list + --set full of the dominant kernels
set -x
python __graft_entry__.py build 2>&1 | tail -2
O=gpurun_out/r02z7
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 --timeout-method thread --durations=10 2>&1 | tail -22 > $O/pytest_gpu.txt
tail -4 $O/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
timeout 1500 python bench.py > $O/bench.json 2> $O/bench.err
tail -c 300 $O/bench.json
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2>> $O/bench.err
timeout 900 python bench.py --partitioned --no-e2e --no-big --no-next > $O/bench_partitioned.json 2>> $O/bench.err
timeout 1500 python bench.py --strong --side 272 --steps 3 --warmup 3 --no-e2e > $O/bench_strong_c5.json 2>> $O/bench.err
timeout 600 python profiles/r02p/trace_c3.py $O/trace_c3.txt > /dev/null 2>&1
python profiles/r02p/analyze_trace.py $O/trace_c3.txt k_tag > $O/trace_summary.txt
B="python bench.py --steps 1 --warmup 1 --no-next --no-e2e --no-cpu-baseline --no-big"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $B > /dev/null 2>&1
python profiles/summarize_launches.py $O/launches.csv $O/launches_summary.csv | head -40
for KS in k_spmv_sell:40 k_update:40 k_small_warp:5 k_num_large_list:1 k_mid_warp:2 k_sym_large:1 k_tail:1 k_level0:1 k_tag:1 k_group_unique:1 k_sell_fill:1; do
  K=${KS%%:*}; S=${KS##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 -o $O/full_$K $B > $O/full_$K.log 2>&1
  ncu -i $O/full_$K.ncu-rep --page raw --csv > $O/full_${K}_raw.csv 2>/dev/null
done
python profiles/summarize_full.py $O > $O/summary.txt
cat $O/summary.txt | head -200
rm -f $O/*.ncu-rep
