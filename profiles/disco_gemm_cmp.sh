# DISCO channel-mix GEMM kernel choice: SPH_DISCO_ALO=0 (BK=16, bn 128/256) vs 1 (BK=32 A_lo-in-TMEM, bn 64/128)
mkdir -p gpurun_out
python -m pytest tests/test_decoder_gpu.py tests/test_disco_gpu.py -x -q > gpurun_out/t_dgemm.log 2>&1; tail -3 gpurun_out/t_dgemm.log
for m in 0 1; do for w in disco decoder; do
SPH_DISCO_ALO=$m python bench.py --workload $w --steps 10 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('alo $m', '$w', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['roofline']['per_kernel_ms'].items()})"
done; done
