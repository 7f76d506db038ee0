# r02x (2): source-level profile of k_num_large_list (stall samples and executed instructions)
set -x
python __graft_entry__.py build 2>&1 | tail -1
mkdir -p gpurun_out/r02x
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-big --no-next"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_num_large_list -s 1 -c 1 -o gpurun_out/r02x/large $B > /dev/null 2>&1
ncu -i gpurun_out/r02x/large.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r02x/src_large.csv 2>/dev/null
gzip -f gpurun_out/r02x/src_large.csv
rm -f gpurun_out/r02x/*.ncu-rep
