#!/bin/bash
# Developer tool: relink libnwb200.so with only weno.cu recompiled under extra
# defines (the default build's other objects reused): variants/<name>.so
#   tools/weno_variant.sh <name> -DNWB_WENO_MINB=4 ...
set -e
NAME=$1; shift
B=build/nwb200
NVCC=${NVCC:-nvcc}
FLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -Xcompiler -O3 --expt-relaxed-constexpr -I paper_2103_06080_b200/csrc -I include"
mkdir -p variants/$NAME.obj
$NVCC $FLAGS "$@" -Xptxas -v -c paper_2103_06080_b200/csrc/weno.cu -o variants/$NAME.obj/weno.o 2>&1 | grep -A2 "${KFILTER:-k_weno_x2IfLi32ELb1}" | grep -E "registers|spill" || true
OBJS=$(ls $B/*.o | grep -v '/weno.o')
$NVCC -gencode arch=compute_100a,code=sm_100a -shared -o variants/$NAME.so $OBJS variants/$NAME.obj/weno.o -lcudart
echo variants/$NAME.so
