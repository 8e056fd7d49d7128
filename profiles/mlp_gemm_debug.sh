# cfg4 MLP GEMMs: full vs no epilogue (SPH_GEMM_DEBUG=1) vs no MMA (4) -- timing only
for d in 0 1 4 5; do
SPH_GEMM_DEBUG=$d timeout 300 python bench.py --workload block --steps 5 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); pk=d['roofline']['per_kernel_ms']; print('dbg $d', {k: round(pk[k],3) for k in ('gemm_mlp1','gemm_mlp2','gemm_disco_mix','gemm_spectral_mix')})"
done
