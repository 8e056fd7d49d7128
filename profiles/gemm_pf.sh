# Legendre GEMM data-tile L2 prefetch distance (SPH_GEMM_PF k-blocks) at cfg2
for PF in 0 2 4 8; do echo -n "PF=$PF "; SPH_GEMM_PF=$PF timeout 120 python profiles/gemm_modes.py 2>&1 | tail -2 | head -1; done
