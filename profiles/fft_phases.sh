# forward fold FFT phase costs at cfg2 (SPH_FFT_DEBUG: 0 full, 1 no store, 2 no phase B/store, 6 loads only)
for D in 0 1 2 6; do echo -n "dbg=$D "; SPH_FFT_DEBUG=$D timeout 120 python profiles/gemm_modes.py 2>&1 | tail -2 | head -1; done
