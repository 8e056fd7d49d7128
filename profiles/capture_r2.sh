#!/bin/bash
# Round-2 evidence capture on the GPU box (1 GPU, run from the repo root):
#   1. the default bench line (exits 0 without ncu)             -> gpurun_out/bench_default.jsonl
#   2. ncu launch list of the same bench command (SHT + DISCO)  -> gpurun_out/launches_bench.csv
#   3. ncu --set full + tensor-pipe counters of the SHT kernels -> gpurun_out/sht_full.ncu-rep
#   4. ncu --set full of the DISCO band kernel and mix GEMM     -> gpurun_out/disco_full.ncu-rep
mkdir -p gpurun_out
TM=sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tensor_subpipe_hmma.sum,sm__inst_executed_pipe_tc.sum,sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
timeout 900 python bench.py > gpurun_out/bench_default.jsonl 2> gpurun_out/bench_default.err
echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e \
    > gpurun_out/ncu_launches.log 2>&1
echo "launches rc=$?"
timeout 900 ncu --set full --metrics $TM --clock-control none --import-source on \
    -k regex:"fft4_|gemm_tf32x3" -c 4 -o gpurun_out/sht_full python profiles/prof_sht.py 1024 1 \
    > gpurun_out/ncu_sht_full.log 2>&1
echo "sht full rc=$?"
timeout 900 ncu --set full --metrics $TM --clock-control none --import-source on \
    -k regex:"disco_band2|gemm_tf32x3" -c 2 -o gpurun_out/disco_full python bench.py --workload disco --steps 1 \
    --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_disco_full.log 2>&1
echo "disco full rc=$?"
