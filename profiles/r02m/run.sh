# r02m: small-row numeric pass reads the symbolic pass's (fine block, child) per sorted key;
# static SELL pattern for the post-coarsening fine solve; bench --strong (C5 at N=1, gloo N=2 run)
set -x
python __graft_entry__.py build 2>&1 | tail -2
mkdir -p gpurun_out/r02m
export AGIPC_SKIP_FULL_CONFIGS=1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_comm_gpu.py tests/test_dist_gpu.py -q -x --timeout 600 --timeout-method thread 2>&1 | tail -5
for i in 1 2; do
  timeout 900 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-big > gpurun_out/r02m/bench$i.json 2>> gpurun_out/r02m/bench.err
done
python - <<'PY'
import json
for i in (1, 2):
    try:
        d = json.loads(open(f"gpurun_out/r02m/bench{i}.json").read().strip().splitlines()[-1])
    except Exception as e:
        print("bench", i, "failed", e); continue
    print({k: d.get(k) for k in ("value", "ms_per_step", "pcg_iters_per_s")}, d["roofline"]["frac"], d.get("phase_ms_per_step"))
    print("next:", d.get("next_rows", {}).get("post_coarsening_pcg"))
PY
timeout 1500 python bench.py --strong --side 272 --steps 3 --warmup 3 --no-e2e > gpurun_out/r02m/bench_strong1.json 2>> gpurun_out/r02m/bench.err
tail -c 1500 gpurun_out/r02m/bench_strong1.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29613 \
  bench.py --strong --side 64 --backend gloo --steps 3 --warmup 3 --no-e2e > gpurun_out/r02m/bench_strong2_gloo.json 2>> gpurun_out/r02m/bench.err
tail -c 1200 gpurun_out/r02m/bench_strong2_gloo.json
tail -5 gpurun_out/r02m/bench.err
timeout 900 python profiles/r02n/probe_c5.py > gpurun_out/r02m/probe_c5.txt 2>&1; tail -12 gpurun_out/r02m/probe_c5.txt
