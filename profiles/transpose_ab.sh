#!/bin/bash
# C_int <-> reference-layout transposes: current build vs libsphgpu_old.so (one field per CTA, one load in flight)
cd "$(dirname "$0")/.."
timeout -s KILL 600 python -m pytest -q -x -m gpu tests/test_sht_gpu.py tests/test_sht_shapes_gpu.py tests/test_baseline_configs_gpu.py tests/test_cpp_shim_gpu.py 2>&1 | tail -2
run() {
  local lab=$1; shift
  env "$@" timeout -s KILL 300 python bench.py --workload sht --steps 10 --no-cpu --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['reference_layout']; print('$lab', round(d['ms_per_step'],3), round(r['ms_per_step'],3), {a: round(b,3) for a, b in r['per_kernel_ms'].items() if 'dense' in a})"
}
for rep in 1 2; do
  run "current " SPH_FFT_DEBUG=0
  run "previous" SPH_LIBSPHGPU=$PWD/paper_2507_12144_b200/libsphgpu_old.so
done
