#!/usr/bin/env bash
# Build the reference package (Python + its Cython kernel) into oracle/_ref/ from the
# read-only sources under /root/reference.  oracle/_ref is git-ignored but travels to
# the GPU box with gpurun snapshots; it is used ONLY as the CPU checker and as the
# `bench.py --impl reference` / cpu_baseline arm.  Never imported by the product.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC=/root/reference/pkg
[ -d "$SRC" ] || { echo "reference not present ($SRC); keeping existing oracle/_ref"; exit 0; }
TMP="$(mktemp -d)"
cp -r "$SRC" "$TMP/pkg" && chmod -R u+w "$TMP/pkg"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$HERE/_ref" --upgrade "$TMP/pkg" >/dev/null
rm -rf "$TMP"
python - <<PY
import sys; sys.path.insert(0, "$HERE/_ref")
import tritransfer; assert tritransfer.kernel_backend == "compiled", tritransfer.kernel_backend
print("oracle/_ref: tritransfer", tritransfer.__version__, "backend", tritransfer.kernel_backend)
PY
