# vectorised row-store epilogue: tests + cfg4 block bench
timeout 900 python -m pytest tests/test_block_gpu.py tests/test_sht_gpu.py tests/test_disco_gpu.py tests/test_decoder_gpu.py tests/test_consumers_gpu.py -x -q 2>&1 | tail -1
for i in 1 2; do timeout 300 python bench.py --workload block --steps 10 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); pk=d['roofline']['per_kernel_ms']; print('block', round(d['ms_per_step'],3), {k: round(pk[k],3) for k in ('gemm_mlp1','gemm_mlp2','gemm_spectral_mix','gemm_disco_mix')})"; done
