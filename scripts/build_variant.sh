#!/bin/bash
# Dev A/B: build libfsg.so variants with extra nvcc defines into
# paper_2206_01683_b200/ab/<name>.so (select at run time with FSG_LIB=...).
#   scripts/build_variant.sh <name> [-DMACRO=V ...]      (current tree)
#   scripts/build_variant.sh <name> --rev <git-rev>       (a committed tree)
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
name=$1; shift
SRC=$ROOT/paper_2206_01683_b200/csrc
if [ "${1:-}" = "--rev" ]; then
  tmp=$(mktemp -d); git -C "$ROOT" archive "$2" paper_2206_01683_b200/csrc include | tar -x -C "$tmp"
  SRC=$tmp/paper_2206_01683_b200/csrc; shift 2
fi
OUT=$ROOT/paper_2206_01683_b200/ab; mkdir -p $OUT/obj_$name
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 -ccbin /usr/bin/g++ $*"
nvcc $F -c $SRC/fsg_kernels_fp32.cu -o $OUT/obj_$name/k32.o &
nvcc $F --fmad=false -c $SRC/fsg_kernels_fp64.cu -o $OUT/obj_$name/k64.o &
nvcc $F -c $SRC/fsg_session.cu -o $OUT/obj_$name/s.o &
[ -f $SRC/fsg_skin.cu ] && nvcc $F --fmad=false -c $SRC/fsg_skin.cu -o $OUT/obj_$name/sk.o &
[ -f $SRC/fsg_drag.cu ] && nvcc $F --fmad=false -c $SRC/fsg_drag.cu -o $OUT/obj_$name/dr.o &
[ -f $SRC/fsg_dyn.cu ] && nvcc $F --fmad=false -c $SRC/fsg_dyn.cu -o $OUT/obj_$name/dy.o &
[ -f $SRC/fsg_io.cpp ] && g++ -std=c++17 -O2 -fPIC -ffp-contract=off -c $SRC/fsg_io.cpp -o $OUT/obj_$name/io.o &
g++ -std=c++17 -O2 -fPIC -ffp-contract=off -c $SRC/fsg_follower.cpp -o $OUT/obj_$name/f.o &
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/$name.so $OUT/obj_$name/*.o -cudart static
rm -rf $OUT/obj_$name
echo built $OUT/$name.so
