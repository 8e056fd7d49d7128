#!/bin/bash
# distributed SHT round trip (configs[4], 721x1440, 512 channels) at 4 GPUs: channel-chunk
# pipelining (SPH_DIST_CHUNKS) x NCCL CTA budget (SPH_NCCL_MAX_CTAS = SMs left to NCCL)
cd "$(dirname "$0")/.."
for D in 4x1 2x2; do
for CH in 1 2 4 8; do
  for CT in 16 32; do
    r=$(SPH_DIST_CHUNKS=$CH SPH_NCCL_MAX_CTAS=$CT timeout -s KILL 300 python bench.py --gpus 4 --workload dist_sht \
        --decomp $D --steps 10 2>/dev/null | tail -1 | \
        python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['domain_decomposed']['sht_roundtrip']; print(round(r['ms_per_step'],3), round(r.get('strong_scaling_eff',0),3))")
    echo "decomp $D chunks $CH nccl_ctas $CT : $r"
  done
done
done
