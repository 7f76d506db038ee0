# r02b (2): static K1 schedule, one-rank all-reduce skip, mirror positions precomputed
set -x
python __graft_entry__.py build 2>&1 | tail -2
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q --durations=10 2>&1 | tail -30 > gpurun_out/r02b2_tests.txt
cat gpurun_out/r02b2_tests.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-next --no-e2e --no-cpu-baseline > gpurun_out/r02b2_bench.json 2> gpurun_out/r02b2_bench.err
tail -3 gpurun_out/r02b2_bench.err; cat gpurun_out/r02b2_bench.json | head -c 3000
timeout 600 python bench.py --partitioned --steps 5 --warmup 3 --no-e2e > gpurun_out/r02b2_part.json 2> gpurun_out/r02b2_part.err
tail -5 gpurun_out/r02b2_part.err; cat gpurun_out/r02b2_part.json | head -c 2000
