#!/bin/bash
# DISCO band kernel: S stored straight from registers (SPH_DISCO_BAND_DIRECT=1) vs staged
# through shared memory
cd "$(dirname "$0")/.."
timeout -s KILL 900 python -m pytest -q -x -m gpu tests/test_disco_gpu.py tests/test_baseline_configs_gpu.py tests/test_decoder_gpu.py tests/test_block_gpu.py 2>&1 | tail -2
SPH_DISCO_BAND_DIRECT=0 timeout -s KILL 900 python -m pytest -q -x -m gpu tests/test_disco_gpu.py 2>&1 | tail -1
run() {
  local lab=$1 w=$2; shift 2
  env "$@" timeout -s KILL 300 python bench.py --workload $w --steps 10 --no-cpu --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['roofline']['per_kernel_ms']; print('$lab $w', round(d['ms_per_step'],3), {a: round(b,3) for a, b in k.items() if 'band' in a or 'mix' in a})"
}
for rep in 1 2; do
  for w in disco decoder; do
    run "direct" $w SPH_DISCO_BAND_DIRECT=1
    run "staged" $w SPH_DISCO_BAND_DIRECT=0
  done
done
