#!/bin/bash
# fused SHT ring transforms: CTA size 256 vs 128 (SPH_FFT_FOLD_THREADS / SPH_FFT_UNFOLD_THREADS)
cd "$(dirname "$0")/.."
SPH_FFT_FOLD_THREADS=128 SPH_FFT_UNFOLD_THREADS=128 timeout -s KILL 600 python -m pytest -q -x -m gpu tests/test_sht_gpu.py tests/test_sht_shapes_gpu.py tests/test_fft_gpu.py 2>&1 | tail -3
for rep in 1 2; do
for cfg in "256 256" "128 256" "256 128" "128 128"; do
  set -- $cfg
  SPH_FFT_FOLD_THREADS=$1 SPH_FFT_UNFOLD_THREADS=$2 timeout -s KILL 300 python bench.py --workload sht --steps 10 --no-cpu --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['roofline']['per_kernel_ms']; print('fold $1 unfold $2', round(d['ms_per_step'],3), {a: round(b,3) for a, b in k.items() if 'fft' in a})"
done
done
