# distributed SHT 2x1 (cfg5) under NCCL channel / protocol settings
for E in "" "NCCL_MIN_NCHANNELS=16" "NCCL_MIN_NCHANNELS=32" "NCCL_PROTO=Simple" "NCCL_MIN_NCHANNELS=32 NCCL_PROTO=Simple" "NCCL_NCHANNELS_PER_NET_PEER=32 NCCL_MIN_NCHANNELS=32 NCCL_MAX_NCHANNELS=64"; do
  echo "env: $E"
  env $E timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29611 bench.py --workload dist_sht --steps 5 --warmup 3 --decomp 2x1 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3))"
done
