#!/usr/bin/env bash
# Build oracle/_ref/dropin_driver: oracle/dropin_driver.cpp (the INTEGRATION.md
# C++ binding) linked against the reference's own sources, compiled where they
# lie under /root/reference (never copied), and against the product library
# paper_2007_06048_b200/libminimod_b200.so (rpath: $ORIGIN/../../paper_2007_06048_b200).
# Test infrastructure only; the binary travels to the GPU box with the tree.
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
root="$(cd "$here/.." && pwd)"
ref="${MINIMOD_REFERENCE:-/root/reference}/proj/core"
if [ ! -d "$ref" ]; then
    echo "build_dropin: $ref not present, skipping (the prebuilt binary is used if any)" >&2
    exit 0
fi
json_dir="$(python - <<'PY'
import glob, os, site
c = []
for sp in site.getsitepackages():
    c += glob.glob(os.path.join(sp, "include", "cudnn_frontend", "thirdparty", "nlohmann"))
print(c[0] if c else "")
PY
)"
[ -n "$json_dir" ] || { echo "build_dropin: nlohmann/json.hpp not found" >&2; exit 1; }
mkdir -p "$here/_ref"
g++ -O3 -DNDEBUG -std=gnu++20 -I"$ref/include" -I"$json_dir" -I"$root/include" \
    "$ref/src/stencil.cpp" "$ref/src/grid.cpp" "$ref/src/model.cpp" \
    "$ref/src/source.cpp" "$ref/src/driver.cpp" "$ref/src/propagator.cpp" \
    "$here/dropin_driver.cpp" -o "$here/_ref/dropin_driver.tmp" \
    -L"$root/paper_2007_06048_b200" -lminimod_b200 \
    -Wl,-rpath,'$ORIGIN/../../paper_2007_06048_b200' -lpthread
mv "$here/_ref/dropin_driver.tmp" "$here/_ref/dropin_driver"
echo "build_dropin: built $here/_ref/dropin_driver"
