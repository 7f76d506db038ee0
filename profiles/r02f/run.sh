# r02f: A/B of the large-row kernels, flat refine, C4 PCG breakdown, ncu of C4 SpMV + flat SpMV
set -x
python __graft_entry__.py build 2>&1 | tail -2
mkdir -p gpurun_out/r02f
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -k "assemble or large or reproducible or c4 or full_size" 2>&1 | tail -3
for V in 0 1; do AGIPC_LARGE_DIRECT=$V timeout 300 python profiles/r02f/probe.py c3; done > gpurun_out/r02f/probe_c3.jsonl 2> gpurun_out/r02f/probe.err
cat gpurun_out/r02f/probe_c3.jsonl
timeout 300 python profiles/r02f/probe.py c4 > gpurun_out/r02f/probe_c4.jsonl 2>> gpurun_out/r02f/probe.err
L2P=0 timeout 300 python profiles/r02f/probe.py c4 >> gpurun_out/r02f/probe_c4.jsonl 2>> gpurun_out/r02f/probe.err
cat gpurun_out/r02f/probe_c4.jsonl; tail -5 gpurun_out/r02f/probe.err
timeout 600 ncu --set full --clock-control none -k regex:k_spmv_sell -s 20 -c 1 -o gpurun_out/r02f/c4_spmv python profiles/r02f/probe.py c4 > /dev/null 2>&1
ncu -i gpurun_out/r02f/c4_spmv.ncu-rep --page raw --csv > gpurun_out/r02f/full_c4_spmv_raw.csv 2>/dev/null
timeout 600 ncu --set full --clock-control none -k regex:k_spmv_flat -s 2 -c 1 -o gpurun_out/r02f/flat python profiles/r02f/probe.py c3 > /dev/null 2>&1
ncu -i gpurun_out/r02f/flat.ncu-rep --page raw --csv > gpurun_out/r02f/full_flat_raw.csv 2>/dev/null
timeout 600 ncu --set full --clock-control none -k regex:k_num_large_fact -s 3 -c 1 -o gpurun_out/r02f/fact python profiles/r02f/probe.py c3 > /dev/null 2>&1
ncu -i gpurun_out/r02f/fact.ncu-rep --page raw --csv > gpurun_out/r02f/full_fact_raw.csv 2>/dev/null
python profiles/summarize_full.py gpurun_out/r02f
