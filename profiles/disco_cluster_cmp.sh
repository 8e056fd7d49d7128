# cfg3 DISCO mix GEMM under table-multicast cluster sizes (SPH_GEMM_CLUSTER)
for c in 1 2 4 1 2 4; do SPH_GEMM_CLUSTER=$c timeout 300 python bench.py --workload disco --steps 10 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cluster $c', round(d['ms_per_step'],3), round(d['roofline']['per_kernel_ms']['gemm_disco_mix'],3))"; done
