#!/bin/bash
# e2e (pinned host -> device -> host) round trip: PCIe ceiling and chunk size sweep
cd "$(dirname "$0")/.."
timeout -s KILL 120 python profiles/pcie_probe.py
for c in 16 32 64 128; do
  timeout -s KILL 600 python bench.py --workload sht --steps 3 --no-cpu --chunk $c 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('chunk $c', round(e['value']), 'fields/s', round(e['ms_per_step'],2), 'ms', round(8.505e3/e['ms_per_step'],1), 'GB/s both ways')"
done
