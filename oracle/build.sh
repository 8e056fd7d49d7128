#!/usr/bin/env bash
# TEST INFRASTRUCTURE: build the C restatement oracle (oracle/liboracle.so) and, where
# /root/reference exists, the reference driver (oracle/_ref/libsphref.so).
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
out="$here/liboracle.so"
if [ ! "$out" -nt "$here/sphere_oracle.c" ] || [ "${FORCE:-0}" = 1 ]; then
  gcc -std=c99 -O2 -fPIC -shared -Wall -Wextra "$here/sphere_oracle.c" -lm -o "$out.tmp"
  mv "$out.tmp" "$out"
  echo "built $out"
fi
"$here/build_ref.sh"
