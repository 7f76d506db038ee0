# r02w: interim capture -- full GPU suite (C4/C5 full size, sanitizers), smoke, full bench, reference arm
set -x
python __graft_entry__.py build 2>&1 | tail -2
mkdir -p gpurun_out/r02w
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 --timeout-method thread --durations=10 2>&1 | tail -25 > gpurun_out/r02w/pytest_gpu.txt
tail -20 gpurun_out/r02w/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02w/smoke.txt 2>&1; tail -2 gpurun_out/r02w/smoke.txt
timeout 1500 python bench.py > gpurun_out/r02w/bench.json 2> gpurun_out/r02w/bench.err
tail -c 600 gpurun_out/r02w/bench.json
