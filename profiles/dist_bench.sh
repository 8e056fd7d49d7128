#!/bin/bash
# cfg5 strong scaling: distributed SHT / DISCO at 721x1440, 512 channels, over the GPUs of
# this box (1x1 on one GPU is T1).  Usage: bash profiles/dist_bench.sh > gpurun_out/dist.jsonl
N=$(nvidia-smi -L | wc -l)
for W in dist_sht dist_disco; do
  timeout 600 python bench.py --workload $W --steps 5 --warmup 3 --decomp 1x1 2>/dev/null | tail -1
  for D in 2x1 1x2 2x2 4x1 1x4; do
    P=$(( ${D%x*} * ${D#*x} ))
    [ $P -le $N ] || continue
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 \
      --master-port $((29600 + P)) bench.py --workload $W --steps 5 --warmup 3 --decomp $D 2>/dev/null | tail -1
  done
done
