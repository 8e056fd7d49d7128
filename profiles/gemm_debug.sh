#!/bin/bash
# GEMM bottleneck isolation: per-tile k-block intervals with parts of the kernel disabled
# (SPH_GEMM_DEBUG bits, see gemm_tc.cu).  Usage (GPU box): bash profiles/gemm_debug.sh
for D in ${DBGS:-0 1 2 3 4 7 8 15}; do
  mkdir -p gpurun_out/dbg$D
  SPH_GEMM_DEBUG=$D SPH_GEMM_TRACE=gpurun_out/dbg$D timeout 120 python profiles/prof_sht.py 1024 1 > /dev/null 2>&1
  echo "dbg=$D"; python profiles/gemm_tiles.py gpurun_out/dbg$D/gemm_tiles_gemm_legendre_fwd.txt gpurun_out/dbg$D/gemm_tiles_gemm_legendre_inv.txt
done
