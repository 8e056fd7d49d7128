#!/bin/bash
# GEMM epilogue hands the TMEM accumulator back before its last chunk's staging / stores
# (current) vs after (libsphgpu_ref.so)
cd "$(dirname "$0")/.."
timeout -s KILL 900 python -m pytest -q -x -m gpu tests/test_sht_gpu.py tests/test_sht_shapes_gpu.py tests/test_disco_gpu.py tests/test_block_gpu.py tests/test_baseline_configs_gpu.py 2>&1 | tail -1
run() {
  local lab=$1 w=$2; shift 2
  env "$@" timeout -s KILL 300 python bench.py --workload $w --steps 10 --no-cpu --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lab $w', round(d['ms_per_step'],3), {a: round(b,3) for a, b in d['roofline']['per_kernel_ms'].items() if 'gemm' in a})"
}
for rep in 1 2; do
  for w in sht disco_t block; do
    run "early" $w SPH_FFT_DEBUG=0
    run "ref  " $w SPH_LIBSPHGPU=$PWD/paper_2507_12144_b200/libsphgpu_ref.so
  done
done
