#!/bin/bash
# Phase times of finalize_kernel (B = 70, one matrix) from a -DSKYRX_FIN_PROFILE build.
set -e
cd "$(dirname "$0")/.."
python -m paper_2602_13509_b200.build >/dev/null
mkdir -p build/fprof
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr \
  -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -prec-div=true -prec-sqrt=true -ftz=false \
  -DSKYRX_FIN_PROFILE "$@" -I include -c paper_2602_13509_b200/csrc/stats.cu -o build/fprof/stats.o
objs=$(ls build/obj/*.o | grep -v '/stats.o$')
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o build/fprof/libskyrx_b200.so \
  $objs build/fprof/stats.o
SKYRX_LIB=build/fprof/libskyrx_b200.so python - <<'PY'
import ctypes, os, sys, torch, numpy as np
sys.path.insert(0, '.')
from paper_2602_13509_b200 import _lib
lib = _lib.load(os.environ['SKYRX_LIB'])
import paper_2602_13509_b200 as P
from paper_2602_13509_b200.synth import Scene
L, S, B = 16384, 900, int(os.environ.get('BANDS', 70))
sc = Scene(4000, S, B, 5)
raw = sc.generate(0, L)
d, c = torch.from_numpy(sc.dark).cuda(), torch.from_numpy(sc.coeff).cuda()
g = torch.ones(L, dtype=torch.float32, device='cuda')
plan = P.DetectPlan(L, S, B)
plan.run(0, raw, d, c, g, gain_const=1.0)
for _ in range(3):
    plan.ds.finalize()
torch.cuda.synchronize()
buf = (ctypes.c_longlong * 12)()
lib.skyrx_fin_profile(buf)
t = np.array(buf[:7], dtype=np.float64)
names = ['moments+sigma+trace', 'cholesky', 'W=L^-1', 'copy W', 'sigma_inv', 'wf']
print({n: int(t[i + 1] - t[i]) for i, n in enumerate(names)}, 'total cycles', int(t[6] - t[0]),
      'wide blocked: panel / trailing cycles (all calls)', buf[8], buf[9])
PY
