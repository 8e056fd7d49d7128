#!/bin/bash
# DISCO forward mix GEMM: default tiles (cfg3 c_out 256: bn 256 BK 16; decoder c_out 64:
# bn 64 A_lo kernel) vs the bn = 192 CTA-pair kernel (SPH_DISCO_MIX_BN=192)
cd "$(dirname "$0")/.."
SPH_DISCO_MIX_BN=192 timeout -s KILL 600 python -m pytest -q -x -m gpu tests/test_disco_gpu.py tests/test_baseline_configs_gpu.py tests/test_decoder_gpu.py tests/test_block_gpu.py 2>&1 | tail -2
run() {
  local lab=$1 w=$2; shift 2
  env "$@" timeout -s KILL 300 python bench.py --workload $w --steps 10 --no-cpu --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lab $w', round(d['ms_per_step'],3), {a: round(b,3) for a, b in d['roofline']['per_kernel_ms'].items()})"
}
for rep in 1 2; do
  for w in disco decoder block; do
    run "default" $w SPH_FFT_DEBUG=0
    run "bn192  " $w SPH_DISCO_MIX_BN=192
  done
done
