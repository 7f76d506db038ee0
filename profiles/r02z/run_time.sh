# wall time of the default bench line (what the driver runs) and of the reference arm
mkdir -p gpurun_out/r02z8
python __graft_entry__.py build 2>&1 | tail -1
t0=$(date +%s); timeout 1500 python bench.py > gpurun_out/r02z8/bench.json 2> gpurun_out/r02z8/bench.err; t1=$(date +%s); echo "bench wall $((t1-t0)) s"
t0=$(date +%s); timeout 900 python bench.py --impl reference > gpurun_out/r02z8/ref.json 2> gpurun_out/r02z8/ref.err; t1=$(date +%s); echo "reference wall $((t1-t0)) s"
python -c "import json; d=json.loads(open('gpurun_out/r02z8/bench.json').read().strip().splitlines()[-1]); print(d['value'], d['pcg_iters_per_s'], d['roofline']['frac'])"
