# MLP1 epilogue: vectorised row stores (SPH_MLP_ROW_TMA=0) vs TMA-store (default)
timeout 600 python -m pytest tests/test_block_gpu.py tests/test_sht_gpu.py tests/test_disco_gpu.py -x -q 2>&1 | tail -1
for v in 0 1 0 1; do SPH_MLP_ROW_TMA=$v timeout 300 python bench.py --workload block --steps 10 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); pk=d['roofline']['per_kernel_ms']; print('row_tma $v', round(d['ms_per_step'],3), round(pk['gemm_mlp1'],3))"; done
