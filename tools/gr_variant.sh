#!/bin/bash
# Time gram_raw built with extra -D flags (e.g. -DSKYRX_GR_PROFILE, or experiment macros):
#   bash tools/gr_variant.sh -DSOME_FLAG
set -e
cd "$(dirname "$0")/.."
python -m paper_2602_13509_b200.build >/dev/null
mkdir -p build/var
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr \
  -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -prec-div=true -prec-sqrt=true -ftz=false \
  "$@" -I include -c paper_2602_13509_b200/csrc/gram_raw.cu -o build/var/gram_raw.o
objs=$(ls build/obj/*.o | grep -v '/gram_raw.o$')
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o build/var/libskyrx_b200.so \
  $objs build/var/gram_raw.o
SKYRX_LIB=build/var/libskyrx_b200.so python - <<'PY'
import os, sys, torch
sys.path.insert(0, '.')
from paper_2602_13509_b200 import _lib
_lib.load(os.environ['SKYRX_LIB'])
import paper_2602_13509_b200 as P
from paper_2602_13509_b200.synth import Scene
L, S, B = 16384, 900, 70
sc = Scene(4000, S, B, 5)
raw = sc.generate(0, L)
d, c = torch.from_numpy(sc.dark).cuda(), torch.from_numpy(sc.coeff).cuda()
g = torch.ones(L, dtype=torch.float32, device='cuda')
plan = P.DetectPlan(L, S, B)
fn = lambda: plan.run(0, raw, d, c, g, gain_const=1.0)
fn(); torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10): fn()
b.record(); torch.cuda.synchronize()
print(sys.argv, 'stats_ms', a.elapsed_time(b) / 10)
PY
