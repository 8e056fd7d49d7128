#!/bin/bash
# distributed SHT pack / unpack: flattened payload tables + batched loads (current) vs
# libsphgpu_old.so (chained payload lookups), cfg5 at the box's GPU count
cd "$(dirname "$0")/.."
N=$(nvidia-smi -L | wc -l)
timeout -s KILL 1200 python -m pytest tests/test_dist.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
run() {
  local lab=$1; shift
  env "$@" timeout -s KILL 600 python bench.py --gpus $N --workload dist_sht --steps 10 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read())['domain_decomposed']; s=d['sht_roundtrip']; print('$lab', d['decomposition'], 'sht', round(s['ms_per_step'],3), 't1', round(s['t1_ms'],3), {a: round(b,3) for a, b in s['per_kernel_ms_rank0'].items() if 'dist' in a}, 'disco', round(d['disco']['ms_per_step'],3))"
}
for rep in 1 2; do
  run "current" SPH_FFT_DEBUG=0
  run "old    " SPH_LIBSPHGPU=$PWD/paper_2507_12144_b200/libsphgpu_old.so
done
