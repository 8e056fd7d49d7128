#!/bin/bash
# C_int <-> dense transposes: 2 fields per CTA sharing the index math (SPH_TR_FIELDS=2) vs 1
cd "$(dirname "$0")/.."
timeout -s KILL 900 python -m pytest -q -x -m gpu tests/test_sht_gpu.py tests/test_sht_shapes_gpu.py tests/test_baseline_configs_gpu.py tests/test_cpp_shim_gpu.py tests/test_consumers_gpu.py tests/test_block_gpu.py 2>&1 | tail -1
SPH_TR_FIELDS=2 timeout -s KILL 900 python -m pytest -q -x -m gpu tests/test_sht_gpu.py tests/test_sht_shapes_gpu.py 2>&1 | tail -1
run() {
  local lab=$1; shift
  env "$@" timeout -s KILL 300 python bench.py --workload sht --steps 10 --no-cpu --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['reference_layout']; print('$lab', round(r['ms_per_step'],3), {a: round(b,3) for a, b in r['per_kernel_ms'].items() if 'dense' in a})"
}
for rep in 1 2 3; do
  run "fields=2" SPH_TR_FIELDS=2
  run "default " SPH_TR_FIELDS=0
done
