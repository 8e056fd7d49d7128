# GEMM pipeline stage width: SPH_GEMM_KS=1 (one 32-wide atom per stage) vs 2 (two atoms:
# half the barrier / fence / commit rounds)
mkdir -p gpurun_out
for k in 2; do SPH_GEMM_KS=$k timeout 900 python -m pytest tests/test_sht_gpu.py tests/test_disco_gpu.py tests/test_decoder_gpu.py tests/test_block_gpu.py tests/test_sht_shapes_gpu.py -x -q 2>&1 | tail -2; done
for k in 1 2; do for w in sht decoder disco; do
SPH_GEMM_KS=$k timeout 300 python bench.py --workload $w --steps 10 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ks $k', '$w', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['roofline']['per_kernel_ms'].items() if k.startswith('gemm')})"
done; done
