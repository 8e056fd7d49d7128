#!/bin/bash
# DISCO-side evidence on the GPU box (run from the repo root):
#   1. bench lines for the disco / decoder / disco_t / block workloads (exit 0 without ncu)
#   2. ncu launch list of the disco bench command
#   3. ncu --set full of the band kernel, the mix GEMM and the decoder's upsample kernel
set -e
mkdir -p gpurun_out
: > gpurun_out/bench_other_workloads.jsonl
for w in disco decoder disco_t block; do
  timeout 600 python bench.py --workload $w --steps 10 >> gpurun_out/bench_other_workloads.jsonl 2>> gpurun_out/bench_other.err
done
tail -4 gpurun_out/bench_other_workloads.jsonl | cut -c1-200
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
    --log-file gpurun_out/launches_disco.csv python bench.py --workload disco --steps 2 --warmup 3 --no-cpu --no-e2e \
    > gpurun_out/ncu_launches_disco.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"disco_band2|gemm_tf32x3" -c 2 -o gpurun_out/disco_full python bench.py --workload disco --steps 1 --warmup 3 --no-cpu --no-e2e \
    > gpurun_out/ncu_disco_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"fourier_upsample|gemm_tf32x3" -c 2 -o gpurun_out/decoder_full python bench.py --workload decoder --steps 1 --warmup 3 --no-cpu --no-e2e \
    > gpurun_out/ncu_decoder_full.log 2>&1
echo capture-ok
