"""Summarise an ncu --set full report (.ncu-rep) into a small JSON for profiles/.

    python profiles/ncu_summary.py gpurun_out/x.ncu-rep profiles/r1/x_summary.json [name=regex ...]

Per kernel: duration, DRAM bytes, throughput percentages, occupancy limits and the top
warp-stall reasons (pc sampling).  name=regex pairs map ncu kernel names to the
library's profiler tags (e.g. fft_fwd_fold=fft4_fold_kernel).
"""
import csv
import io
import json
import re
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__bytes.sum.per_second", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_tensor_subpipe_hmma.sum", "sm__inst_executed_pipe_tc.sum",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
    "launch__grid_size", "launch__block_size", "sm__cycles_elapsed.avg.per_second",
]


def main():
    rep, out = sys.argv[1], sys.argv[2]
    names = dict(a.split("=", 1) for a in sys.argv[3:])
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    res = []
    for row in rows[2:]:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        kn = d.get("Kernel Name", "")
        tag = next((t for t, rx in names.items() if re.search(rx, kn)), None)
        e = {"kernel": tag or kn[:80], "ncu_kernel": kn[:160]}
        for k in KEYS:
            if k in d and d[k] not in ("", "n/a"):
                e[k] = f"{d[k]} {u.get(k, '')}".strip()
        stalls = []
        for k, v in d.items():
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
                try:
                    stalls.append((k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v)))
                except ValueError:
                    pass
        tot = sum(v for _, v in stalls) or 1.0
        stalls.sort(key=lambda x: -x[1])
        e["top_stalls_pct"] = {k: round(100 * v / tot, 1) for k, v in stalls[:6]}
        res.append(e)
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1)[:3000])


if __name__ == "__main__":
    main()
