#!/bin/bash
# GeLU as 0.5 x (1 + erf(x / sqrt 2)) (libsphgpu_erf.so, -DSPH_GELU_ERF) vs the erfc form
cd "$(dirname "$0")/.."
SPH_LIBSPHGPU=$PWD/paper_2507_12144_b200/libsphgpu_erf.so timeout -s KILL 600 python -m pytest -q -x -m gpu tests/test_block_gpu.py tests/test_baseline_configs_gpu.py 2>&1 | tail -2
run() {
  local lab=$1; shift
  env "$@" timeout -s KILL 300 python bench.py --workload block --steps 10 --no-cpu --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['roofline']['per_kernel_ms']; print('$lab', round(d['ms_per_step'],3), {a: round(b,3) for a, b in k.items() if 'mlp' in a})"
}
for rep in 1 2; do
  run "erfc" SPH_FFT_DEBUG=0
  run "erf " SPH_LIBSPHGPU=$PWD/paper_2507_12144_b200/libsphgpu_erf.so
done
