#!/bin/bash
# forward Legendre GEMM E/O operand map: 512-byte inner runs (default) vs 1 KB (SPH_GEMM_AQUAD_1K=1)
cd "$(dirname "$0")/.."
SPH_GEMM_AQUAD_1K=1 timeout -s KILL 600 python -m pytest -q -x -m gpu tests/test_sht_gpu.py tests/test_sht_shapes_gpu.py tests/test_baseline_configs_gpu.py 2>&1 | tail -2
run() {
  local lab=$1; shift
  env "$@" timeout -s KILL 300 python bench.py --workload sht --steps 10 --no-cpu --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lab', round(d['ms_per_step'],3), {a: round(b,3) for a, b in d['roofline']['per_kernel_ms'].items()})"
}
for rep in 1 2 3; do
  run "512B" SPH_GEMM_AQUAD_1K=0
  run "1KB " SPH_GEMM_AQUAD_1K=1
done
