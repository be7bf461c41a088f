#!/bin/bash
# Phase cycles of finalize_panel_kernel (matrix 0) from a -DSKYRX_FIN_PROFILE build.
set -e
cd "$(dirname "$0")/.."
python -m paper_2602_13509_b200.build >/dev/null
mkdir -p build/fpprof
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr \
  -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -prec-div=true -prec-sqrt=true -ftz=false \
  -DSKYRX_FIN_PROFILE "$@" -I include -c paper_2602_13509_b200/csrc/finalize_panel.cu -o build/fpprof/fp.o
objs=$(ls build/obj/*.o | grep -v '/finalize_panel.o$')
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o build/fpprof/libskyrx_b200.so \
  $objs build/fpprof/fp.o
SKYRX_LIB=build/fpprof/libskyrx_b200.so python - <<'PY'
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
    buf = (ctypes.c_longlong * 16)()
    for _ in range(3):
        ctypes.memset(buf, 0, ctypes.sizeof(buf))
        lib.skyrx_fp_profile(buf)  # read to keep the symbol live
        ds.finalize()
    torch.cuda.synchronize()
    lib.skyrx_fp_profile(buf)
    t = np.array(buf[:], dtype=np.float64)
    names = ['moments+sigma+trace', 'factor+inverse', 'sigma_inv', 'outputs']
    ph = {nm: int(t[i + 1] - t[i]) for i, nm in enumerate(names)}
    # accumulators add up over the 3 calls and over lanes-0 of the warps that ran them
    print(B, ph, 'total', int(t[4] - t[0]), '| warp0 chol', int(t[5] / 3), 'wpanel', int(t[6] / 3),
          '| Rtrail (15 warps sum)', int(t[7] / 3), 'Atrail', int(t[8] / 3), flush=True)
PY
