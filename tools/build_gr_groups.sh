#!/bin/bash
# gram_raw epilogue-group variants: tools/build_gr_groups.sh G -> tools/_var/gr_g$G/libskyrx_b200.so
set -e
cd "$(dirname "$0")/.."
G=$1
mkdir -p tools/_var/gr_g$G
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr \
  -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -prec-div=true -prec-sqrt=true -ftz=false \
  -DGRX_EPI_GROUPS=$G -I include -c paper_2602_13509_b200/csrc/gram_raw.cu -o tools/_var/gr_g$G/gram_raw.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o tools/_var/gr_g$G/libskyrx_b200.so \
  $(ls build/obj/*.o | grep -v '/gram_raw.o$') tools/_var/gr_g$G/gram_raw.o
