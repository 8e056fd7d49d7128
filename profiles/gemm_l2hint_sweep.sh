#!/bin/bash
# Legendre GEMM L2 cache-policy hints (SPH_GEMM_L2HINT: 1 evict-first output stores, 2 evict-last
# table loads, 3 both) on the cfg2 round trip, 1 GPU; per-kernel ms from the bench's live timing
cd "$(dirname "$0")/.."
for H in 0 1 2 3 0; do
  SPH_GEMM_L2HINT=$H timeout -s KILL 300 python bench.py --workload sht --steps 20 --no-cpu --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('l2hint $H', round(d['ms_per_step'],3), {k: round(v,3) for k, v in d['roofline']['per_kernel_ms'].items()})"
done
