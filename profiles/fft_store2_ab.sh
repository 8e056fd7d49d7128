#!/bin/bash
# fold store phase: two-row threads (default) vs one thread per (m, field) (SPH_FFT_STORE2=1);
# packed fp32x2 FFT math (current build) vs the scalar build (libsphgpu_old.so)
cd "$(dirname "$0")/.."
SPH_FFT_STORE2=1 timeout -s KILL 600 python -m pytest -q -x -m gpu tests/test_sht_gpu.py tests/test_sht_shapes_gpu.py 2>&1 | tail -2
run() {  # label, env...
  local lab=$1; shift
  env "$@" timeout -s KILL 300 python bench.py --workload sht --steps 10 --no-cpu --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['roofline']['per_kernel_ms']; print('$lab', round(d['ms_per_step'],3), {a: round(b,3) for a, b in k.items() if 'fft' in a})"
}
for rep in 1 2 3; do
  run "packed store2=0" SPH_FFT_STORE2=0
  run "packed store2=1" SPH_FFT_STORE2=1
  run "scalar(old lib)" SPH_LIBSPHGPU=$PWD/paper_2507_12144_b200/libsphgpu_old.so
done
