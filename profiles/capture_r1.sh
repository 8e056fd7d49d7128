#!/bin/bash
# Round-1 evidence capture on the GPU box (run from the repo root):
#   1. bench.py default run (exits 0 without ncu)  -> gpurun_out/bench_default.jsonl
#   2. ncu launch list of the same bench command   -> gpurun_out/launches_bench.csv
#   3. ncu --set full of one launch of each hot kernel at the bench workload
set -e
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_default.jsonl 2> gpurun_out/bench_default.err
tail -1 gpurun_out/bench_default.jsonl
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e \
    > gpurun_out/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"fft4_|gemm_tf32x3" -c 4 -o gpurun_out/sht_full python profiles/prof_sht.py 1024 1 \
    > gpurun_out/ncu_full.log 2>&1
echo capture-ok
