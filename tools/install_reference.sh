#!/usr/bin/env bash
# Install the UNMODIFIED reference package (locmax, /root/reference/pkg) into
# baseline/_ref for bench.py's reference arm and cpu_baseline leg.
# Offline: no index; numpy is already in the image, so dependency resolution
# is skipped (--no-deps).  The build writes into its source tree, so it runs
# from a copy under /tmp (/root/reference is read-only).
# baseline/_ref is git-ignored but travels to the GPU box with gpurun.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC="${1:-/root/reference/pkg}"
TMP="$(mktemp -d /tmp/locmax_src.XXXXXX)"
cp -r "$SRC"/. "$TMP"/
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" "$TMP"
rm -rf "$TMP"
PYTHONPATH="$ROOT/baseline/_ref" python -c "import locmax, sys; print('installed', locmax.__file__)"
