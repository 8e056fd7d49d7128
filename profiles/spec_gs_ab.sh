#!/bin/bash
# spectral gather / scatter with batched row-offset loads (current) vs the previous build
cd "$(dirname "$0")/.."
timeout -s KILL 900 python -m pytest -q -x -m gpu tests/test_block_gpu.py tests/test_baseline_configs_gpu.py -k "block or spectral or cfg4" 2>&1 | tail -1
run() {
  local lab=$1; shift
  env "$@" timeout -s KILL 300 python bench.py --workload block --steps 10 --no-cpu --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lab', round(d['ms_per_step'],3), {a: round(b,3) for a, b in d['roofline']['per_kernel_ms'].items() if 'spectral' in a})"
}
for rep in 1 2 3; do
  run "batched" SPH_FFT_DEBUG=0
  run "ref    " SPH_LIBSPHGPU=$PWD/paper_2507_12144_b200/libsphgpu_ref.so
done
