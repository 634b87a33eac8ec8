#!/bin/bash
# Development aid: libtobf with extra conv_tc.cu defines into
# scripts/_probe_libs/libtobf_<name>.so (use with TOBF_LIB=...).
# usage: scripts/build_variant_lib.sh NAME -DFOO=1 ...
set -e
cd "$(dirname "$0")/.."
name=$1; shift
python -c "from paper_2107_09789_b200 import build_native; build_native.build()"
mkdir -p scripts/_probe_libs/obj_$name
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude \
  -Ipaper_2107_09789_b200/csrc "$@" -c paper_2107_09789_b200/csrc/conv_tc.cu -o scripts/_probe_libs/obj_$name/conv_tc.o
objs=$(ls build/native/*.o | grep -v conv_tc.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o scripts/_probe_libs/libtobf_$name.so $objs scripts/_probe_libs/obj_$name/conv_tc.o
echo built scripts/_probe_libs/libtobf_$name.so
