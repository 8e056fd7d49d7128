#!/usr/bin/env bash
# TEST INFRASTRUCTURE: compile the UNMODIFIED reference headers (spheretk) behind the
# C-ABI driver oracle/ref_driver.cpp into oracle/_ref/libsphref.so.  Reference
# Release flags (proj/CMakeLists.txt:8-14): -std=c++20 -O3 -DNDEBUG.
# Only runs where /root/reference exists (the dev container); the built .so travels
# to the GPU box with the repo snapshot (git-ignored, not gpurun-ignored).
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
ref="${SPHERE_REF_INCLUDE:-/root/reference/proj/include}"
# model.hpp -> sfd.hpp:18 needs nlohmann <json.hpp>; the image vendors one (cudnn_frontend).
json="${SPHERE_JSON_INCLUDE:-$(python3 -c 'import site,os;print(os.path.join(site.getsitepackages()[0],"include/cudnn_frontend/thirdparty/nlohmann"))' 2>/dev/null)}"
if [ ! -d "$ref/sphere" ]; then
  echo "build_ref.sh: reference headers not found at $ref (skipping)" >&2
  exit 0
fi
mkdir -p "$here/_ref"
out="$here/_ref/libsphref.so"
if [ "$out" -nt "$here/ref_driver.cpp" ] && [ "${FORCE:-0}" != 1 ]; then exit 0; fi
g++ -std=c++20 -O3 -DNDEBUG -fPIC -shared -pthread -Wall -Wextra \
    -I"$ref" -I"$json" "$here/ref_driver.cpp" -o "$out.tmp"
mv "$out.tmp" "$out"
echo "built $out"
