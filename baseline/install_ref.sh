#!/bin/sh
# Install the UNMODIFIED reference (gnnsim, /root/reference/pkg) into
# baseline/_ref -- git-ignored, but not gpurun-ignored, so it travels to the
# GPU box.  The build writes into its source tree, so it runs from a copy.
# Dependencies (numpy, numba) are already in the image: --no-deps.
# The reference's own test-suite is placed beside it (baseline/_ref/gnnsim_tests)
# for tests/test_gnnsim_dropin_gpu.py, which runs it against our CUDA kernels.
set -e
HERE=$(cd "$(dirname "$0")" && pwd)
SRC=${GNNSIM_SRC:-/root/reference/pkg}
PY=${PYTHON:-python}
[ -d "$SRC" ] || { echo "reference not found at $SRC" >&2; exit 1; }
TMP=$(mktemp -d)
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"
rm -rf "$HERE/_ref"
"$PY" -m pip install -q --no-index --no-build-isolation --no-deps \
    --find-links /opt/wheelhouse --target "$HERE/_ref" "$TMP/pkg"
cp -r "$SRC/tests" "$HERE/_ref/gnnsim_tests"
echo "installed gnnsim into $HERE/_ref"
