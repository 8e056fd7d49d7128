#!/bin/bash
# DISCO adjoint band kernel: __launch_bounds__(128, 4) (128 registers, 4 CTAs/SM) vs the
# previous build (154 registers, 3 CTAs/SM)
cd "$(dirname "$0")/.."
timeout -s KILL 600 python -m pytest -q -x -m gpu tests/test_disco_gpu.py tests/test_baseline_configs_gpu.py 2>&1 | tail -2
run() {
  local lab=$1; shift
  env "$@" timeout -s KILL 300 python bench.py --workload disco_t --steps 10 --no-cpu --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lab', round(d['ms_per_step'],3), {a: round(b,3) for a, b in d['roofline']['per_kernel_ms'].items()})"
}
for rep in 1 2; do
  run "current" SPH_FFT_DEBUG=0
  run "old    " SPH_LIBSPHGPU=$PWD/paper_2507_12144_b200/libsphgpu_old.so
done
