#!/bin/bash
# Instrumented build of the library (tools/timeline.py): -DCSB_TIMELINE.
set -e
cd "$(dirname "$0")/.."
C=paper_2003_08011_b200/csrc
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --shared \
  -Xcompiler -fPIC -DCSB_TIMELINE -I include -I $C $C/cstress_b200.cu $C/synth.cpp $C/model_io.cpp \
  -o tools/libcstress_b200_tl.so -lpthread -ldl 2>&1 | grep -v "^$" || true
ls -la tools/libcstress_b200_tl.so
