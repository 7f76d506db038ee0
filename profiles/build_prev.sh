#!/bin/bash
# Build variants/prev/libagipc.so from the committed (HEAD) version of the given csrc files, for
# A/B runs of uncommitted changes.  Usage: bash profiles/build_prev.sh [files, default assemble.cu]
set -e
SRCS=${1:-assemble.cu}
cd "$(dirname "$0")/.."
python __graft_entry__.py build > /dev/null
mkdir -p variants/prev/src
FLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -cudart static -Iinclude -Ipaper_2605_04773_b200/csrc"
OBJS=""
for o in paper_2605_04773_b200/build/*.o; do
  b=$(basename $o .o)
  if [[ " $SRCS " == *" $b.cu "* ]]; then
    git show HEAD:paper_2605_04773_b200/csrc/$b.cu > variants/prev/src/$b.cu
    nvcc $FLAGS -c variants/prev/src/$b.cu -o variants/prev/$b.o
    OBJS="$OBJS variants/prev/$b.o"
  else
    OBJS="$OBJS $o"
  fi
done
nvcc -shared -gencode arch=compute_100a,code=sm_100a -cudart static -o variants/prev/libagipc.so $OBJS -ldl
echo variants/prev/libagipc.so
