"""Post-process a profiles/final_r2.sh run (gpurun_out/) into profiles/r2/final/.

    python profiles/process_final_r2.py

Copies the suite log, bench line and reference arm, summarises the ncu captures
(profiles/ncu_summary.py) with the library's kernel tags, refreshes
profiles/ncu_traffic_sht.json (the `traffic` / tensor-pipe figures bench.py reports) and
writes the launch-list summary.
"""
import collections
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
DST = os.path.join(ROOT, "profiles", "r2", "final")


def gb(s):
    v, u = s.split()
    return float(v) * {"Tbyte": 1e12, "Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}[u]


def summarise(rep, out, names, tags=None):
    subprocess.run([sys.executable, os.path.join(ROOT, "profiles", "ncu_summary.py"), rep, out] + names,
                   check=True, capture_output=True)
    d = json.load(open(out))
    if tags:
        for e, t in zip(d, tags):
            e["kernel"] = t
    for e in d:
        if "gemm_tf32x3" in e["kernel"]:
            e["kernel"] = "gemm_disco_mix"
    json.dump(d, open(out, "w"), indent=1)
    return {e["kernel"]: e for e in d}


def main():
    os.makedirs(DST, exist_ok=True)
    for f in ("gpu_suite_final.log", "bench_default.jsonl", "bench_reference.jsonl", "final_r2.log"):
        shutil.copy(os.path.join(OUT, f), DST)
    shutil.copy(os.path.join(OUT, "launches_bench.csv"), os.path.join(DST, "launches_bench_default.csv"))
    sht = summarise(os.path.join(OUT, "sht_full.ncu-rep"), os.path.join(DST, "ncu_full_sht_f1024_summary.json"),
                    ["fft_fwd_fold=fft4_fold_kernel", "fft_inv_unfold=fft4_unfold_kernel"],
                    ["fft_fwd_fold", "gemm_legendre_fwd", "gemm_legendre_inv", "fft_inv_unfold"])
    dis = summarise(os.path.join(OUT, "disco_full.ncu-rep"), os.path.join(DST, "ncu_full_disco_cfg3_summary.json"),
                    ["disco_band=disco_band2"])
    tp = "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic_sht.json")
    t = json.load(open(tpath))
    for k in t["dram_bytes_per_launch"]:
        t["dram_bytes_per_launch"][k] = gb(sht[k]["dram__bytes_read.sum"]) + gb(sht[k]["dram__bytes_write.sum"])
    dd = t["by_workload"]["disco"]["dram_bytes_per_launch"]
    for k in dd:
        dd[k] = gb(dis[k]["dram__bytes_read.sum"]) + gb(dis[k]["dram__bytes_write.sum"])
    t["tensor_pipe_active_pct"] = {"gemm_legendre_fwd": sht["gemm_legendre_fwd"][tp],
                                   "gemm_legendre_inv": sht["gemm_legendre_inv"][tp],
                                   "gemm_disco_mix": dis["gemm_disco_mix"][tp]}
    json.dump(t, open(tpath, "w"), indent=1)
    rows = [r for r in csv.reader(open(os.path.join(DST, "launches_bench_default.csv"))) if len(r) > 5]
    hdr, rows = rows[0], rows[1:]
    ki, mi, vi, ui = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    scale = {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows:
        if r[mi] == "gpu__time_duration.sum":
            tot[r[ki]] += float(r[vi].replace(",", "")) * scale[r[ui]]
            cnt[r[ki]] += 1
    total = sum(tot.values())
    lines = ["ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised) of",
             "python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e (round 2 final, 1x B200; the first 600 launches",
             "of the default line): kernel, launches, total ms, share", ""]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        lines.append(f"{v:9.3f} ms {cnt[k]:4d}x {100 * v / total:6.1f}%  {k[:90]}")
    open(os.path.join(DST, "launches_bench_default_summary.txt"), "w").write("\n".join(lines) + "\n")
    line = json.loads(open(os.path.join(DST, "bench_default.jsonl")).read().strip().splitlines()[-1])
    print("value", round(line["value"]), "ms", round(line["ms_per_step"], 3),
          {k: round(v, 3) for k, v in line["roofline"]["per_kernel_ms"].items()})
    print("reference layout", round(line["reference_layout"]["ms_per_step"], 3), "disco",
          round(line["disco"]["ms_per_step"], 3), "block", round(line["block"]["ms_per_step"], 3),
          "cfg1", line["cfg1"]["ms_per_step"], "e2e", round(line["e2e"]["value"]), "cpu",
          line["cpu_baseline"]["value"], "clocks", line["clocks"])


if __name__ == "__main__":
    main()
