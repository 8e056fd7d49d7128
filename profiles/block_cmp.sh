python -m pytest tests/test_block_gpu.py -x -q 2>&1 | tail -2
PYTHONPATH=. python profiles/block_probe.py
python bench.py --workload block --steps 10 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('block', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['roofline']['per_kernel_ms'].items()})"
