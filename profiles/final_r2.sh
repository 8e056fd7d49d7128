#!/bin/bash
# Final round-2 evidence on one B200 (run from the repo root): GPU suite, reference arm,
# then capture_r2.sh (bench line, ncu launch list, ncu --set full of the SHT / DISCO kernels)
mkdir -p gpurun_out
timeout -s KILL 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_suite_final.log 2>&1
echo "gpu suite rc=$?"; tail -3 gpurun_out/gpu_suite_final.log
timeout -s KILL 900 python bench.py --impl reference > gpurun_out/bench_reference.jsonl 2> gpurun_out/bench_reference.err
echo "reference arm rc=$?"
bash profiles/capture_r2.sh
