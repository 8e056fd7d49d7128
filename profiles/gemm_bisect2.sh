for D in 16 32 48; do echo "dbg=$D"; SPH_GEMM_DEBUG=$D NLATS="361" bash profiles/gemm_bisect.sh 2>&1 | grep -v watchdog | tail -1; done
