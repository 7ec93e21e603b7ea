#!/usr/bin/env bash
# Compile the reference's own acoustic_iso_cd translation units, exactly as
# they lie under /root/reference (read-only, never copied), together with
# oracle/ref_shim.cpp into oracle/_ref/libminimod_ref.so.  Flags match the
# reference's Release build (-O3 -DNDEBUG -std=gnu++20, no -march: SSE2, no
# FMA).  nlohmann/json (header-only; source.cpp/model.cpp's shot-record and
# model-manifest I/O, which the format tests pin against) comes from the
# image's cudnn_frontend wheel (nlohmann 3.11.3).
# Test infrastructure only.
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
ref="${MINIMOD_REFERENCE:-/root/reference}/proj/core"
if [ ! -d "$ref" ]; then
    echo "build_ref: $ref not present, skipping (prebuilt oracle/_ref is used if any)" >&2
    exit 0
fi
json_dir="$(python - <<'EOF'
import glob, os, site
cands = []
for sp in site.getsitepackages():
    cands += glob.glob(os.path.join(sp, "include", "cudnn_frontend", "thirdparty", "nlohmann"))
print(cands[0] if cands else "")
EOF
)"
if [ -z "$json_dir" ]; then
    echo "build_ref: nlohmann/json.hpp not found; cannot build the reference" >&2
    exit 1
fi
mkdir -p "$here/_ref"
g++ -O3 -DNDEBUG -std=gnu++20 -fPIC -shared \
    -I"$ref/include" -I"$json_dir" \
    "$ref/src/stencil.cpp" "$ref/src/grid.cpp" "$ref/src/model.cpp" \
    "$ref/src/source.cpp" "$ref/src/driver.cpp" "$ref/src/propagator.cpp" \
    "$here/ref_shim.cpp" -o "$here/_ref/libminimod_ref.so.tmp" -lpthread
mv "$here/_ref/libminimod_ref.so.tmp" "$here/_ref/libminimod_ref.so"
echo "build_ref: built $here/_ref/libminimod_ref.so"
