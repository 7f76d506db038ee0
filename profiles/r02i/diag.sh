# diagnostic (not committed): k_small_warp numeric without mirror writes / without own-row value writes
python __graft_entry__.py build 2>&1 | tail -1
mkdir -p gpurun_out/r02j
for D in 0 1 2 3; do
 AGIPC_DBG_SMALL=$D timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_small_warp -c 4 --csv python profiles/r02f/probe.py c3 2>/dev/null | grep -E "k_small_warp" | tail -3 > gpurun_out/r02j/d$D.csv
 echo "== dbg $D"; cat gpurun_out/r02j/d$D.csv | cut -c1-400
done
