python __graft_entry__.py build 2>&1 | tail -1
mkdir -p gpurun_out/r02g
timeout 600 python -m pytest tests/test_dist_gpu.py tests/test_gpu_parity.py -q --timeout 300 --timeout-method thread -k "8-2-5-random or map or assemble_c1 or c4_contact" 2>&1 | grep -v "^  " | tail -40 > gpurun_out/r02g/t2.txt
cat gpurun_out/r02g/t2.txt
