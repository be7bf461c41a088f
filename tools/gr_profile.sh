#!/bin/bash
# Build a gram_raw variant with the per-role wait probes and run tools/gr_profile.py on it.
set -e
cd "$(dirname "$0")/.."
python -m paper_2602_13509_b200.build >/dev/null
mkdir -p build/prof
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr \
  -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -prec-div=true -prec-sqrt=true -ftz=false \
  -DSKYRX_GR_PROFILE "$@" -I include -c paper_2602_13509_b200/csrc/gram_raw.cu -o build/prof/gram_raw.o
objs=$(ls build/obj/*.o | grep -v '/gram_raw.o$')
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o build/prof/libskyrx_b200.so \
  $objs build/prof/gram_raw.o
SKYRX_LIB=build/prof/libskyrx_b200.so python tools/gr_profile.py
