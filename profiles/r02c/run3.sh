# r02c (3): default atomic large rows restored; AGIPC_OPT_DETERMINISTIC path; full gpu suite
set -x
python __graft_entry__.py build 2>&1 | tail -2
mkdir -p gpurun_out/r02c3
timeout 1500 python -m pytest tests -m gpu -q --timeout 400 --timeout-method thread --durations=12 \
   2>&1 | tail -40 > gpurun_out/r02c3/tests.txt
cat gpurun_out/r02c3/tests.txt
timeout 600 python bench.py --steps 10 --warmup 3 --no-next --no-e2e --no-cpu-baseline --no-big > gpurun_out/r02c3/bench.json 2> gpurun_out/r02c3/bench.err
tail -3 gpurun_out/r02c3/bench.err; head -c 2500 gpurun_out/r02c3/bench.json
timeout 600 python bench.py --partitioned --steps 5 --warmup 3 --no-e2e > gpurun_out/r02c3/part.json 2> gpurun_out/r02c3/part.err
tail -3 gpurun_out/r02c3/part.err; head -c 1500 gpurun_out/r02c3/part.json
