set -x
python __graft_entry__.py build 2>&1 | tail -1
bash profiles/ab_libs.sh gpurun_out/r02s3 "base s128m6 s160m5 s96m6"
bash profiles/ab_libs.sh gpurun_out/r02s3s "base s128m6 s160m5 s96m6" AGIPC_NUM_MODE=1
