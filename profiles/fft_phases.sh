# FFT phase costs at cfg2 (SPH_FFT_DEBUG): forward fold 1 no store, 2 no phase B/store, 6 loads only;
# inverse unfold 16 no store, 48 loads only
for D in 0 1 2 6 16 48; do echo -n "dbg=$D "; SPH_FFT_DEBUG=$D timeout 120 python profiles/gemm_modes.py 2>&1 | tail -2 | head -1; done
