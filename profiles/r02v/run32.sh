set -x
python __graft_entry__.py build 2>&1 | tail -1
bash profiles/ab_libs.sh gpurun_out/r02v32 "base l0m6 l0m8 sl16"
