set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc; lscpu | grep "Model name"
python __graft_entry__.py build 2>&1 | tail -2
timeout 1500 python -m pytest tests -x -q -m gpu --durations=15 -s 2>&1 | grep -v "^$" | tail -60 > gpurun_out/r02a_gputest.txt
tail -30 gpurun_out/r02a_gputest.txt
