#!/bin/bash
# A/B build of the library with experiment macros: tools/build_variant.sh NAME -DQX_EXP_... ;
# the result is paper_2505_03307_b200/lib/libqimax_b200_NAME.so, picked with QX_LIB=<path>.
set -e
name=$1; shift
cd "$(dirname "$0")/../paper_2505_03307_b200/csrc"
out=../../build/exp_$name
mkdir -p $out
flags="-O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-Wall,-Wno-unused-function --expt-relaxed-constexpr -Xptxas -v"
for f in store clifford branch dense merge readout partition wide; do
  nvcc $flags "$@" -c $f.cu -o $out/$f.o 2> $out/$f.ptxas.log &
done
wait
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o ../lib/libqimax_b200_$name.so $out/*.o -cudart static
echo built ../lib/libqimax_b200_$name.so
