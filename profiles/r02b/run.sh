# r02b: library-owned NCCL communicator + workspace + ADVICE fixes on one B200
set -x
python __graft_entry__.py build 2>&1 | tail -2
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_comm_gpu.py tests/test_dist_gpu.py tests/test_gpu_parity.py -x -q --durations=8 2>&1 | tail -25 > gpurun_out/r02b_tests.txt
cat gpurun_out/r02b_tests.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-next > gpurun_out/r02b_bench.json 2> gpurun_out/r02b_bench.err
tail -3 gpurun_out/r02b_bench.err; cat gpurun_out/r02b_bench.json | head -c 3000
timeout 600 python bench.py --partitioned --steps 5 --warmup 3 --no-e2e > gpurun_out/r02b_part.json 2> gpurun_out/r02b_part.err
tail -5 gpurun_out/r02b_part.err; cat gpurun_out/r02b_part.json | head -c 2000
