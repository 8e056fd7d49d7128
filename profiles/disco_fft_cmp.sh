python -m pytest tests/test_disco_gpu.py tests/test_fft_gpu.py tests/test_decoder_gpu.py -x -q 2>&1 | tail -2
for w in disco disco_t decoder; do
python bench.py --workload $w --steps 10 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['roofline']['per_kernel_ms'].items()})"
done
