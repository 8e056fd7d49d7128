#!/bin/bash
# distributed SHT round trip at 4x1 on the final tree (in-place stage addressing): channel
# chunks x NCCL CTA budget
cd "$(dirname "$0")/.."
for E in "SPH_NCCL_MAX_CTAS=32" "SPH_NCCL_MAX_CTAS=24" "SPH_NCCL_MAX_CTAS=48"; do
  for CH in 1 2 3 4; do
    r=$(env $E SPH_DIST_CHUNKS=$CH timeout -s KILL 300 python bench.py --gpus 4 --workload dist_sht \
        --decomp 4x1 --steps 10 2>/dev/null | tail -1 | \
        python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['domain_decomposed']; s=r['sht_roundtrip']; print('sht', round(s['ms_per_step'],3), 'disco', round(r['disco']['ms_per_step'],3))")
    echo "$E chunks $CH : $r"
  done
done
