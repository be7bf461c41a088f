#!/bin/bash
# Phase cycles of finalize_small_kernel (one matrix) from a -DSKYRX_FIN_PROFILE build.
set -e
cd "$(dirname "$0")/.."
python -m paper_2602_13509_b200.build >/dev/null
mkdir -p build/fsprof
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr \
  -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -prec-div=true -prec-sqrt=true -ftz=false \
  -DSKYRX_FIN_PROFILE "$@" -I include -c paper_2602_13509_b200/csrc/finalize_small.cu -o build/fsprof/fs.o
objs=$(ls build/obj/*.o | grep -v '/finalize_small.o$')
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o build/fsprof/libskyrx_b200.so \
  $objs build/fsprof/fs.o
SKYRX_LIB=build/fsprof/libskyrx_b200.so python - <<'PY'
import ctypes, os, sys, torch, numpy as np
sys.path.insert(0, '.')
from paper_2602_13509_b200 import _lib
lib = _lib.load(os.environ['SKYRX_LIB'])
import paper_2602_13509_b200 as P
rng = np.random.default_rng(0)
for B in (16, 70, 128):
    n = 100000
    X = rng.standard_normal((4096, B)) @ np.diag(np.linspace(1, 30, B))
    mom = np.concatenate([[float(n)], X.sum(0) * 0, (X.T @ X * (n / 4096)).ravel()])
    ds = P.DeviceStats(B, batch=1)
    ds.moments.copy_(torch.from_numpy(mom))
    for _ in range(3):
        ds.finalize()
    torch.cuda.synchronize()
    buf = (ctypes.c_longlong * 8)()
    lib.skyrx_fs_profile(buf)
    t = np.array(buf[:5], dtype=np.float64)
    names = ['moments+sigma+trace', 'factor+inverse', 'sigma_inv', 'outputs']
    print(B, {n: int(t[i + 1] - t[i]) for i, n in enumerate(names)}, 'total', int(t[4] - t[0]))
PY
