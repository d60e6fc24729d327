"""pytest plugin (``-p gnnsim_cuda_plugin``): run the REFERENCE's own test-suite
(baseline/_ref/gnnsim_tests, installed by baseline/install_ref.sh) with its
operator layer bound to the B200 library (paper_2409_00657_b200._kernels_cuda)
-- the GNNSIM_KERNELS=cuda backend of INTEGRATION.md.  Counts the calls that
reach the CUDA kernels and prints them at the end of the session, so the
caller can check the GPU path really ran."""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(REPO, "baseline", "_ref")
for p in (REPO, REF):
    if p not in sys.path:
        sys.path.insert(0, p)

import gnnsim.kernels as _gk  # noqa: E402

from paper_2409_00657_b200 import _kernels_cuda as _cuda  # noqa: E402

CALLS = {}


def _counted(name, fn):
    def wrap(*a, **k):
        CALLS[name] = CALLS.get(name, 0) + 1
        return fn(*a, **k)
    wrap.__name__ = name
    return wrap


_cuda.install(_gk)
for _n in ("sample_frontier", "feature_rows", "pick_k_smallest", "sbm_edges"):
    setattr(_gk, _n, _counted(_n, getattr(_gk, _n)))


def pytest_sessionfinish(session, exitstatus):
    print("\nGNNSIM_CUDA_CALLS " + " ".join(f"{k}={v}" for k, v in sorted(CALLS.items())))
