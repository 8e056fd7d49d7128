#!/bin/bash
# distributed C_int unpack with two fields per CTA: NCCL parity + 2x1 timing
cd "$(dirname "$0")/.."
timeout -s KILL 1200 python -m pytest -q -x -m gpu tests/test_dist.py 2>&1 | tail -1
for rep in 1 2; do
timeout -s KILL 600 python bench.py --gpus 2 --workload dist_sht --steps 10 2>/dev/null | tail -1 | \
  python -c "import json,sys; d=json.loads(sys.stdin.read())['domain_decomposed']; s=d['sht_roundtrip']; print('dist 2x1 sht', round(s['ms_per_step'],3), 't1', round(s['t1_ms'],3), {a: round(b,3) for a, b in s['per_kernel_ms_rank0'].items() if 'dist' in a})"
done
