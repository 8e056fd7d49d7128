# forward fold FFT CTA order: ring quads fastest (default) vs field groups fastest
SPH_FFT_FY_FAST=1 timeout 600 python -m pytest tests/test_sht_gpu.py tests/test_fft_gpu.py -x -q 2>&1 | tail -1
for v in 0 1 0 1; do
SPH_FFT_FY_FAST=$v timeout 300 python bench.py --steps 10 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fy_fast $v', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['roofline']['per_kernel_ms'].items()})"
done
