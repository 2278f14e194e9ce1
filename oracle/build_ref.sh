#!/usr/bin/env bash
# Build the UNMODIFIED reference verifier into oracle/_ref/ (test infrastructure
# only). Sources are compiled where they lie under /root/reference/proj; nothing
# is copied into this repo. Needs: g++ (C++20), the runtime libgmp.so.10, and
# nlohmann/json (only present in this image under the venv's cudnn_frontend
# headers; symlinked into oracle/_ref/vendor). The output .so is git-ignored
# but travels to the GPU box with the gpurun snapshot (libgmp.so.10 is in the
# same image there).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF="${POLYCERT_REF:-/root/reference/proj}"
OUT="$HERE/_ref"
mkdir -p "$OUT/vendor"
if [ ! -d "$REF" ]; then
  echo "build_ref: reference not present at $REF (GPU box?) — skipping" >&2
  exit 0
fi
JSON="$(python3 -c 'import site,os;print(next(p for p in [os.path.join(s,"include/cudnn_frontend/thirdparty/nlohmann/json.hpp") for s in site.getsitepackages()] if os.path.exists(p)))' 2>/dev/null || true)"
if [ -z "$JSON" ]; then echo "build_ref: nlohmann/json.hpp not found" >&2; exit 1; fi
ln -sf "$JSON" "$OUT/vendor/json.hpp"
GMP="$(ls /lib/x86_64-linux-gnu/libgmp.so.10 /usr/lib/x86_64-linux-gnu/libgmp.so.10 2>/dev/null | head -1)"
# -O3 -DNDEBUG = the reference's CMake Release build (proj/CMakeLists.txt:8-10).
# -ffp-contract=off: keep the reference's separate multiply/add roundings
# (its CMake build uses no -march, so x86-64 has no FMA to contract into).
CXXFLAGS="-std=c++20 -O3 -DNDEBUG -fPIC -ffp-contract=off -w -I$HERE/shim -I$OUT/vendor -I$REF/include"
g++ $CXXFLAGS -shared -o "$OUT/libpolycert_ref.so" \
  "$HERE/ref_driver.cpp" "$REF/src/decimal.cpp" "$REF/src/gen.cpp" "$REF/src/model_io.cpp" \
  "$GMP" -lpthread
echo "built $OUT/libpolycert_ref.so"
