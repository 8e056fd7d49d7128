#!/bin/bash
# A/B of two builds of libsphgpu.so on one box (SPH_LIBSPHGPU), alternating, cfg2 + cfg3
cd "$(dirname "$0")/.."
for L in paper_2507_12144_b200/libsphgpu.so paper_2507_12144_b200/libsphgpu_old.so paper_2507_12144_b200/libsphgpu.so paper_2507_12144_b200/libsphgpu_old.so; do
  for W in sht disco; do
    SPH_LIBSPHGPU=$PWD/$L timeout -s KILL 300 python bench.py --workload $W --steps 10 --no-cpu --no-e2e 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['roofline']['per_kernel_ms']; print('$(basename $L) $W', round(d['ms_per_step'],3), {a: round(b,3) for a, b in k.items() if 'fft' in a})"
  done
done
