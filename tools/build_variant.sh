#!/bin/bash
# Build an experiment variant of libfgs.so that differs in ONE source file: recompile that file with
# extra -D flags and relink with the other objects of the last normal build.
# Usage: bash tools/build_variant.sh NAME SRC.cu "-DFLAG ..."   ->  exp_libs/libfgs_NAME.so
set -e
NAME=$1; SRC=$2; FLAGS=$3
D=paper_2310_08528_b200
mkdir -p exp_libs /tmp/fgs_var_$NAME
NVCC="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC -Xcompiler -O3"
$NVCC $FLAGS -c $D/csrc/$SRC -o /tmp/fgs_var_$NAME/$SRC.o
OBJS=""
for o in $D/build/*.cu.o; do
  if [ "$(basename $o)" = "$SRC.o" ]; then OBJS="$OBJS /tmp/fgs_var_$NAME/$SRC.o"; else OBJS="$OBJS $o"; fi
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -o exp_libs/libfgs_$NAME.so $OBJS -cudart static
echo exp_libs/libfgs_$NAME.so
