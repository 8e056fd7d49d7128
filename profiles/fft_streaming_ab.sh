#!/bin/bash
# SHT ring transforms with streaming cache hints (ld.global.cs input rings, st.global.cs
# output rings; libsphgpu_strm.so built with -DSPH_FFT_STREAMING) vs the default build
cd "$(dirname "$0")/.."
SPH_LIBSPHGPU=$PWD/paper_2507_12144_b200/libsphgpu_strm.so timeout -s KILL 600 python -m pytest -q -x -m gpu tests/test_sht_gpu.py 2>&1 | tail -1
run() {
  local lab=$1; shift
  env "$@" timeout -s KILL 300 python bench.py --workload sht --steps 10 --no-cpu --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lab', round(d['ms_per_step'],3), {a: round(b,3) for a, b in d['roofline']['per_kernel_ms'].items()})"
}
for rep in 1 2 3; do
  run "default  " SPH_FFT_DEBUG=0
  run "streaming" SPH_LIBSPHGPU=$PWD/paper_2507_12144_b200/libsphgpu_strm.so
done
