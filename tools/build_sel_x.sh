#!/bin/bash
# select.cu variants: tools/build_sel_x.sh NAME -DFLAG -> tools/_var/NAME/libskyrx_b200.so
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p tools/_var/$name
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr \
  -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -prec-div=true -prec-sqrt=true -ftz=false \
  "$@" -I include -c paper_2602_13509_b200/csrc/select.cu -o tools/_var/$name/select.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o tools/_var/$name/libskyrx_b200.so \
  $(ls build/obj/*.o | grep -v '/select.o$') tools/_var/$name/select.o
