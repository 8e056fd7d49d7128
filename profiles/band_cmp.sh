mkdir -p gpurun_out
python -m pytest tests/test_decoder_gpu.py tests/test_disco_gpu.py -x -q > gpurun_out/t_band.log 2>&1; tail -3 gpurun_out/t_band.log
for m in 1 2; do for w in disco decoder; do
SPH_DISCO_BAND=$m python bench.py --workload $w --steps 10 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('mode $m', '$w', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['roofline']['per_kernel_ms'].items()})"
done; done
