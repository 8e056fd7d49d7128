#!/bin/bash
# inverse Legendre GEMM: raw table split by the converter in SMEM (default) vs host-split hi/lo tables
cd "$(dirname "$0")/.."
for E in ${SWEEP:-"X=1" "SPH_GEMM_BLO_CONV=0" "X=1" "SPH_GEMM_BLO_CONV=0" "X=1" "SPH_GEMM_BLO_CONV=0"}; do
  env $E timeout -s KILL 300 python bench.py --workload sht --steps 10 --no-cpu --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['roofline']['per_kernel_ms']; print('$E', round(d['ms_per_step'],3), 'fwd', round(k['gemm_legendre_fwd'],3), 'inv', round(k['gemm_legendre_inv'],3))"
done
