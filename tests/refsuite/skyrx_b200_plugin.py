"""pytest plugin: route the reference package through the B200 library BEFORE the
reference's own test modules import it (they bind names at import:
`from skyrx.rx import compute_stats`), like selecting a backend with SKYRX_NO_NUMBA
(_accel.py:21-31).  Used by tests/test_gpu_reference_suite.py; writes the patched
names and the number of C-ABI calls the session made to $SKYRX_B200_PLUGIN_LOG."""

import json
import os

import skyrx  # the reference, from baseline/_ref

import paper_2602_13509_b200 as P
from paper_2602_13509_b200 import _lib

PATCHED = P.install(skyrx)


def pytest_sessionfinish(session, exitstatus):
    log = os.environ.get("SKYRX_B200_PLUGIN_LOG")
    if log:
        with open(log, "w") as fh:
            json.dump({"patched": PATCHED, "capi_calls": _lib.CALLS,
                       "library": str(_lib.load()._name)}, fh)
