#!/bin/bash
# Build a variant of libagipc.so with extra nvcc defines for A/B runs (AGIPC_LIB=<path>).
# Usage: bash profiles/build_variant.sh NAME "-DFOO=1 -DBAR=2" [sources to rebuild, default assemble.cu]
set -e
NAME=$1; DEFS=$2; SRCS=${3:-assemble.cu}
cd "$(dirname "$0")/.."
python __graft_entry__.py build > /dev/null
mkdir -p variants/$NAME
FLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -cudart static -Iinclude"
OBJS=""
for o in paper_2605_04773_b200/build/*.o; do
  b=$(basename $o .o)
  if [[ " $SRCS " == *" $b.cu "* ]]; then
    nvcc $FLAGS $DEFS -c paper_2605_04773_b200/csrc/$b.cu -o variants/$NAME/$b.o
    OBJS="$OBJS variants/$NAME/$b.o"
  else
    OBJS="$OBJS $o"
  fi
done
nvcc -shared -gencode arch=compute_100a,code=sm_100a -cudart static -o variants/$NAME/libagipc.so $OBJS -ldl
echo variants/$NAME/libagipc.so
