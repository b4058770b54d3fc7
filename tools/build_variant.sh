#!/bin/bash
# A/B build of the library with extra -D flags (development tool):
#   tools/build_variant.sh NAME -DFOO=1 ...  ->  tools/var/libcstress_NAME.so
# Only cstress_b200.cu is recompiled; the other objects come from the
# regular build (python -m paper_2003_08011_b200.build).  Run a tool against
# it with CSB_LIB=tools/var/libcstress_NAME.so.
set -e
cd "$(dirname "$0")/.."
NAME=$1; shift
C=paper_2003_08011_b200/csrc
B=paper_2003_08011_b200/build
mkdir -p tools/var
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  -I include -I $C "$@" -c $C/cstress_b200.cu -o tools/var/$NAME.o
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a --shared -Xcompiler -fPIC tools/var/$NAME.o \
  $B/train_f64.cu.o $B/synth.cpp.o $B/model_io.cpp.o -o tools/var/libcstress_$NAME.so -lpthread -ldl
echo tools/var/libcstress_$NAME.so
