#!/bin/bash
# incremental-index transposes / packs: GPU parity (1 and 2 ranks) + timing
cd "$(dirname "$0")/.."
timeout -s KILL 1200 python -m pytest -q -x -m gpu tests/test_sht_gpu.py tests/test_sht_shapes_gpu.py tests/test_baseline_configs_gpu.py tests/test_cpp_shim_gpu.py tests/test_dist.py tests/test_consumers_gpu.py 2>&1 | tail -2
bash profiles/transpose_ab.sh 2>&1 | grep -v passed
timeout -s KILL 600 python bench.py --gpus 2 --workload dist_sht --steps 10 2>/dev/null | tail -1 | \
  python -c "import json,sys; d=json.loads(sys.stdin.read())['domain_decomposed']; s=d['sht_roundtrip']; print('dist 2x1 sht', round(s['ms_per_step'],3), {a: round(b,3) for a, b in s['per_kernel_ms_rank0'].items() if 'dist' in a})"
