#!/bin/bash
# distributed SHT round trip at 4x1: NCCL CTA budget and copy-engine P2P under chunking
cd "$(dirname "$0")/.."
for E in "SPH_NCCL_MAX_CTAS=32" "SPH_NCCL_MAX_CTAS=48" "SPH_NCCL_MAX_CTAS=64" "SPH_NCCL_MAX_CTAS=16 NCCL_P2P_USE_CUDA_MEMCPY=1" "SPH_NCCL_MAX_CTAS=32 NCCL_P2P_USE_CUDA_MEMCPY=1"; do
  for CH in 1 2 3; do
    r=$(env $E SPH_DIST_CHUNKS=$CH timeout -s KILL 300 python bench.py --gpus 4 --workload dist_sht \
        --decomp 4x1 --steps 10 2>/dev/null | tail -1 | \
        python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['domain_decomposed']['sht_roundtrip']; print(round(r['ms_per_step'],3), round(r.get('strong_scaling_eff',0),3))")
    echo "$E chunks $CH : $r"
  done
done
