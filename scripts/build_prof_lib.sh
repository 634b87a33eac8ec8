#!/bin/bash
# Development aid: libtobf with the conv role-timing counters (TOBF_CONV_PROF)
# into scripts/_probe_libs/libtobf_prof.so (use with TOBF_LIB=...).
set -e
cd "$(dirname "$0")/.."
python -c "from paper_2107_09789_b200 import build_native; build_native.build()"
mkdir -p scripts/_probe_libs/obj
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude \
  -Ipaper_2107_09789_b200/csrc -DTOBF_CONV_PROF -c paper_2107_09789_b200/csrc/conv_tc.cu -o scripts/_probe_libs/obj/conv_tc.o
objs=$(ls build/native/*.o | grep -v conv_tc.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o scripts/_probe_libs/libtobf_prof.so $objs scripts/_probe_libs/obj/conv_tc.o
echo built scripts/_probe_libs/libtobf_prof.so
