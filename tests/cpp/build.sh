#!/bin/bash
# Build the C++ drop-in pin program (tests/cpp/shim_pins.cpp) against the UNMODIFIED
# reference headers and libsphgpu.so.  Needs /root/reference (this container); the binary
# lands in tests/cpp/_bin/ (git-ignored, travels to the GPU box with the tree).
set -e
HERE="$(cd "$(dirname "$0")" && pwd)"
ROOT="$(cd "$HERE/../.." && pwd)"
REF="${SPH_REFERENCE_INCLUDE:-/root/reference/proj/include}"
if [ ! -d "$REF" ]; then echo "reference headers not present: skipping shim_pins"; exit 0; fi
mkdir -p "$HERE/_bin"
g++ -std=c++20 -O2 -I"$REF" -I"$ROOT/include" -I/usr/local/cuda/include "$HERE/shim_pins.cpp" \
    -L"$ROOT/paper_2507_12144_b200" -l:libsphgpu.so -L/usr/local/cuda/lib64 -lcudart \
    -Wl,-rpath,'$ORIGIN/../../../paper_2507_12144_b200' -Wl,-rpath,/usr/local/cuda/lib64 \
    -o "$HERE/_bin/shim_pins"
echo "$HERE/_bin/shim_pins"
