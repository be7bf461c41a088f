#!/bin/bash
# build a select experiment variant: tools/build_gr_var.sh <name> -DFLAG...
# -> tools/_var/<name>.so (gpurun ships it; *.so is git-ignored)
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p build/var tools/_var
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr \
  -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -prec-div=true -prec-sqrt=true -ftz=false \
  "$@" -I include -c paper_2602_13509_b200/csrc/select.cu -o build/var/select_$name.o 2>&1 | grep -i error || true
objs=$(ls build/obj/*.o | grep -v '/select.o$')
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o tools/_var/$name.so \
  $objs build/var/select_$name.o
