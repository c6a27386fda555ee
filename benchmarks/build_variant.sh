#!/bin/bash
# build_variant.sh <name> <source.cu> <extra nvcc flags...>: an A/B copy of the library with one
# source recompiled with extra flags -> paper_1804_05038_b200/_lib/libqnmt_b200_<name>.so
# (run with QNMT_LIB_PATH=<that file>)
set -e
name=$1; src=$2; shift 2
here=$(cd "$(dirname "$0")/.." && pwd)
pk=$here/paper_1804_05038_b200
obj=/tmp/qnmt_variant_${name}.o
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC,-fvisibility=hidden \
  -Xptxas -O3 --expt-relaxed-constexpr -I $here/include "$@" -c $pk/csrc/$src -o $obj
objs=$(ls $pk/_lib/obj/*.o | grep -v "/${src%.cu}.o")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $pk/_lib/libqnmt_b200_${name}.so $objs $obj -lcudart_static -lrt -ldl -lpthread
echo built $pk/_lib/libqnmt_b200_${name}.so
