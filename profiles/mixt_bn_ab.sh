#!/bin/bash
# DISCO adjoint mix GEMM (N = c_in K = 576 at cfg3): bn = 192 CTA-pair kernel (exact 3 tiles)
# vs bn = 256 (pads N to 768)
cd "$(dirname "$0")/.."
timeout -s KILL 600 python -m pytest -q -x -m gpu tests/test_disco_gpu.py tests/test_baseline_configs_gpu.py tests/test_block_gpu.py tests/test_decoder_gpu.py 2>&1 | tail -2
run() {
  local lab=$1; shift
  env "$@" timeout -s KILL 300 python bench.py --workload disco_t --steps 10 --no-cpu --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lab', round(d['ms_per_step'],3), {a: round(b,3) for a, b in d['roofline']['per_kernel_ms'].items()})"
}
for rep in 1 2; do
  run "bn192" SPH_FFT_DEBUG=0
  run "bn256" SPH_DISCO_MIXT_BN=256
  run "bn128" SPH_DISCO_MIXT_BN=128
done
