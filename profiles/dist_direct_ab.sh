#!/bin/bash
# distributed SHT with the ring transforms reading / writing the all-to-all stage blocks in
# place (current) vs the box-copy unpack / pack passes (SPH_DIST_BOXCOPY=1)
cd "$(dirname "$0")/.."
N=$(nvidia-smi -L | wc -l)
timeout -s KILL 1500 python -m pytest tests/test_dist.py tests/test_sht_gpu.py tests/test_sht_shapes_gpu.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
run() {
  local lab=$1; shift
  env "$@" timeout -s KILL 600 python bench.py --gpus $N --workload dist_sht --steps 10 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read())['domain_decomposed']; s=d['sht_roundtrip']; print('$lab', d['decomposition'], 'sht', round(s['ms_per_step'],3), 't1', round(s['t1_ms'],3), 'eff', round(s['strong_scaling_eff'],3), {a: round(b,3) for a, b in s['per_kernel_ms_rank0'].items()})"
}
for rep in 1 2; do
  run "direct " SPH_FFT_DEBUG=0
  run "boxcopy" SPH_DIST_BOXCOPY=1
done
