#!/bin/bash
# Legendre GEMM role knock-outs (SPH_GEMM_DEBUG bits; results are WRONG when set, timing only):
# 1 epilogue skips TMEM loads + stores, 2 converter skips its work, 4 no MMAs, 8 no table loads
cd "$(dirname "$0")/.."
for D in 0 1 2 4 3 7 15; do
  SPH_GEMM_DEBUG=$D timeout -s KILL 300 python bench.py --workload sht --steps 10 --no-cpu --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['roofline']['per_kernel_ms']; print('dbg $D', 'fwd', round(k['gemm_legendre_fwd'],3), 'inv', round(k['gemm_legendre_inv'],3))"
done
