#!/usr/bin/env bash
# Install the UNMODIFIED reference package (jointsched, /root/reference/pkg) into baseline/_ref.
# baseline/_ref is git-ignored but not gpurun-ignored: it travels to the GPU box with the repo
# snapshot, where /root/reference does not exist.  Used by the drop-in tests (reference pydantic
# objects through plan_saturn / resolve, validated by the reference's own core.check_plan).
# The build writes egg-info next to the sources, so it installs from a copy under /tmp.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC="${REFERENCE_PKG:-/root/reference/pkg}"
[ -d "$SRC" ] || { echo "reference package not found at $SRC" >&2; exit 1; }
TMP="$(mktemp -d)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --find-links /opt/wheelhouse --no-deps \
    --target "$ROOT/baseline/_ref" "$TMP/pkg" >/dev/null
test -f "$ROOT/baseline/_ref/jointsched/core.py"
echo "installed jointsched into baseline/_ref"
