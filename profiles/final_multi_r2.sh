#!/bin/bash
# Final round-2 multi-GPU evidence on one 4x B200 box (repo root): NCCL parity tests at 2 and
# 4 ranks, then the self-launching bench at N = 2 and N = 4 (field-sharded weak line + the
# cfg5 domain-decomposed record)
mkdir -p gpurun_out
timeout -s KILL 1500 python -m pytest tests/test_dist.py -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_dist_4gpu.log 2>&1
echo "dist suite rc=$?"; tail -3 gpurun_out/gpu_dist_4gpu.log
CUDA_VISIBLE_DEVICES=0,1 timeout -s KILL 900 python bench.py --gpus 2 --no-cpu > gpurun_out/bench_n2.jsonl 2> gpurun_out/bench_n2.err
echo "bench n2 rc=$?"
timeout -s KILL 900 python bench.py --gpus 4 --no-cpu > gpurun_out/bench_n4.jsonl 2> gpurun_out/bench_n4.err
echo "bench n4 rc=$?"
