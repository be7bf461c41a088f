#!/bin/bash
# Stage the reference package and its hot-path test modules under baseline/_ref
# (git-ignored, not gpurun-ignored: travels to the GPU box), for
# tests/test_gpu_reference_suite.py and bench.py's reference arm.  Needs /root/reference
# (this container only).  The package install is the one the task prescribes
# (pip --no-index --target baseline/_ref, from a copy: the build writes into the tree).
set -e
cd "$(dirname "$0")/.."
REF=${REF:-/root/reference/pkg}
[ -d "$REF" ] || { echo "no reference at $REF"; exit 0; }
if [ ! -f baseline/_ref/skyrx/rx.py ]; then
  rm -rf /tmp/skyrx_ref_src && cp -r "$REF" /tmp/skyrx_ref_src
  python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target baseline/_ref /tmp/skyrx_ref_src
fi
mkdir -p baseline/_ref/tests
for f in conftest.py test_rx.py test_calibrate.py test_accel.py test_acceptance.py \
         test_pipeline.py test_datalink.py test_fec.py test_cube.py; do
  cp "$REF/tests/$f" baseline/_ref/tests/
done
echo "staged: $(ls baseline/_ref/tests | tr '\n' ' ')"
