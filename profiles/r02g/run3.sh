python __graft_entry__.py build 2>&1 | tail -1
mkdir -p gpurun_out/r02g
for i in 1 2; do timeout 600 python -m pytest tests/test_dist_gpu.py -q --timeout 300 --timeout-method thread 2>&1 | grep -v "^  " | tail -30; done > gpurun_out/r02g/t3.txt
cat gpurun_out/r02g/t3.txt
