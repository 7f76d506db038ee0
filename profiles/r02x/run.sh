# r02x: source-level profile of the small-row kernels (stall samples and executed instructions)
set -x
python __graft_entry__.py build 2>&1 | tail -1
mkdir -p gpurun_out/r02x
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-big --no-next"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_small_warp -s 4 -c 2 -o gpurun_out/r02x/small $B > /dev/null 2>&1
ncu -i gpurun_out/r02x/small.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r02x/src_small.csv 2>/dev/null
head -5 gpurun_out/r02x/src_small.csv | cut -c1-600
ncu -i gpurun_out/r02x/small.ncu-rep --page raw --csv > gpurun_out/r02x/full_small_raw.csv 2>/dev/null
python profiles/summarize_full.py gpurun_out/r02x
gzip -f gpurun_out/r02x/src_small.csv
rm -f gpurun_out/r02x/*.ncu-rep
