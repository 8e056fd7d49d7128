#!/bin/bash
# inverse ring transform: 512-thread CTAs (16 fields per row, 128-byte EOi runs, 1 CTA/SM)
# vs 256 (8 fields, 2 CTAs/SM)
cd "$(dirname "$0")/.."
SPH_FFT_UNFOLD_THREADS=512 timeout -s KILL 600 python -m pytest -q -x -m gpu tests/test_sht_gpu.py tests/test_sht_shapes_gpu.py 2>&1 | tail -1
run() {
  local lab=$1; shift
  env "$@" timeout -s KILL 300 python bench.py --workload sht --steps 10 --no-cpu --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lab', round(d['ms_per_step'],3), {a: round(b,3) for a, b in d['roofline']['per_kernel_ms'].items() if 'fft' in a})"
}
for rep in 1 2 3; do
  run "256" SPH_FFT_UNFOLD_THREADS=256
  run "512" SPH_FFT_UNFOLD_THREADS=512
done
