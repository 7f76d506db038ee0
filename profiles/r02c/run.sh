# r02c: large-row chunks with deterministic partials (no atomics), mirror positions precomputed,
# k_tail on an ordinary launch with a software grid barrier; parity + bench + launch list
set -x
python __graft_entry__.py build 2>&1 | tail -2
mkdir -p gpurun_out/r02c
export AGIPC_SKIP_FULL_CONFIGS=1
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 --timeout-method thread --durations=10 \
   2>&1 | tail -30 > gpurun_out/r02c/tests.txt
cat gpurun_out/r02c/tests.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-next --no-e2e --no-cpu-baseline --no-big > gpurun_out/r02c/bench.json 2> gpurun_out/r02c/bench.err
tail -3 gpurun_out/r02c/bench.err; head -c 2500 gpurun_out/r02c/bench.json
AGIPC_TAIL_COOP=1 timeout 600 python bench.py --steps 5 --warmup 3 --no-next --no-e2e --no-cpu-baseline --no-big > gpurun_out/r02c/bench_coop.json 2>> gpurun_out/r02c/bench.err
python -c "import json;d=json.load(open('gpurun_out/r02c/bench_coop.json'));print('coop', d['value'], d['phase_ms_per_step'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02c/launches.csv \
  python bench.py --steps 1 --warmup 1 --no-next --no-e2e --no-cpu-baseline --no-big > gpurun_out/r02c/launches_bench.log 2>&1
python profiles/summarize_launches.py gpurun_out/r02c/launches.csv gpurun_out/r02c/launches_summary.csv | head -40
