#!/bin/bash
# NCCL all-to-all bandwidth and the library's distributed SHT round trip under NCCL settings (4 GPUs)
cd "$(dirname "$0")/.."
for E in "X=1" "NCCL_MIN_NCHANNELS=32" "NCCL_MAX_NCHANNELS=64 NCCL_MIN_NCHANNELS=64" "NCCL_PROTO=Simple" "NCCL_NVLS_ENABLE=0" "NCCL_P2P_LEVEL=NVL NCCL_MIN_P2P_NCHANNELS=32" "NCCL_MIN_P2P_NCHANNELS=32 NCCL_MAX_P2P_NCHANNELS=64"; do
  env $E SWEEP_TAG="$E" timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 29611 profiles/a2a_bw.py 2>/dev/null
  env $E timeout 300 python bench.py --gpus 4 --workload dist_sht --steps 10 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('  dist_sht rt ms', round(d['ms_per_step'],3))"
done
