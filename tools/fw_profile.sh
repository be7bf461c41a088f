#!/bin/bash
# Phase cycles of fw_factor_kernel (finalize_wide.cu, B = 270 by default) from a
# -DSKYRX_FW_PROFILE build: left-looking updates / panel factorisations / write-backs.
set -e
cd "$(dirname "$0")/.."
python -m paper_2602_13509_b200.build >/dev/null
mkdir -p build/fwprof
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr \
  -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -prec-div=true -prec-sqrt=true -ftz=false \
  -DSKYRX_FW_PROFILE "$@" -I include -c paper_2602_13509_b200/csrc/finalize_wide.cu -o build/fwprof/finalize_wide.o
objs=$(ls build/obj/*.o | grep -v '/finalize_wide.o$')
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o build/fwprof/libskyrx_b200.so \
  $objs build/fwprof/finalize_wide.o
SKYRX_LIB=build/fwprof/libskyrx_b200.so python - <<'PY'
import ctypes, os, sys, torch, numpy as np
sys.path.insert(0, '.')
from paper_2602_13509_b200 import _lib
lib = _lib.load(os.environ['SKYRX_LIB'])
import paper_2602_13509_b200 as P
B = int(os.environ.get('BANDS', 270))
rng = np.random.default_rng(0)
n = 100000
X = rng.standard_normal((4096, B)) @ np.diag(np.linspace(1, 30, B))
mom = np.concatenate([[float(n)], X.sum(0) * 0, (X.T @ X * (n / 4096)).ravel()])
ds = P.DeviceStats(B, batch=1)
ds.moments.copy_(torch.from_numpy(mom[None]))
ds.finalize()
torch.cuda.synchronize()
buf = (ctypes.c_longlong * 4)()
lib.skyrx_fw_profile(buf)
print(f"B={B} one call: left-looking {buf[0]}  panels {buf[1]}  write-back {buf[2]} cycles")
PY
