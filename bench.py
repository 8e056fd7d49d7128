"""Benchmark of the spherical-operator hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload all|sht|disco|disco_t|block|decoder|dist_sht|dist_disco]

Default (``--workload all``), one JSON line:
  * ``value``: configs[1] -- forward + inverse SHT on the 721x1440 equiangular grid,
    lmax=721 (count) / mmax=720, 256 channels x batch 4 = 1024 fields per GPU; one step =
    sht_inverse(sht_forward(x)) over those fields.  For N > 1 every rank transforms its own
    1024 fields (batch/channel sharding, no data-path collective) -> "scaling": "weak";
    value = all fields / max-over-ranks time.
  * ``disco``: configs[2] -- DISCO 721x1440 eq -> 360x720 Gaussian, Morlet K=9, cutoff
    3*pi/360, 64 -> 256 channels, batch 4 per GPU (output fields/s), with its own roofline,
    e2e and CPU baseline.
  * ``domain_decomposed`` (N > 1): configs[4] -- the paper's lat/lon decomposition through
    the library's NCCL path (csrc/dist.cu): distributed SHT + inverse SHT round trip and
    distributed DISCO (-> 360x720 Gaussian) at 721x1440, 512 channels, batch 1, polar x
    azimuth = N x 1, strong scaling against the same problem on one GPU of the same run.

``python bench.py --gpus N`` launches N ranks itself (torchrun, 127.0.0.1) when it is not
already running under torchrun.

``--impl reference`` times the reference's own CPU implementation (the unmodified
headers compiled into oracle/_ref/libsphref.so; the C restatement if that is absent) on
the host cores of rank 0, a bounded sample of the same workload per step.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

NLAT, NLON, LMAX, MMAX = 721, 1440, 721, 720
BATCH, CHANNELS = 4, 256
FIELDS = BATCH * CHANNELS
METRIC = "SHT+ISHT & DISCO-conv fields/sec at 721\u00d71440, % of roofline, at 1/2/4/8 GPUs"  # BASELINE.json metric
UNIT = "fields/s"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], p["bf16_tflops"], p.get("bf16_tflops_sustained", p["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock + clock-event (throttle) reasons sampled DURING the timed region.

    NVML (nvidia_ml_py) polled every 5 ms from a thread, so even a ~100 ms timed region
    gets ~20 samples; falls back to `nvidia-smi -lms 50` when NVML is unavailable."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4}

    def __init__(self, index: int):
        self.index = index
        self.sm, self.mx, self.reasons = [], None, set()
        self.stop = threading.Event()
        self.proc = None
        self.t = None

    def _nvml_handle(self):
        import pynvml
        pynvml.nvmlInit()
        try:  # map the CUDA device to the NVML device through its PCI bus id
            import torch
            pr = torch.cuda.get_device_properties(self.index)
            bus = "%08x:%02x:%02x.0" % (pr.pci_domain_id, pr.pci_bus_id, pr.pci_device_id)
            return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.index)

    def _poll_nvml(self, nv, h):
        while not self.stop.is_set():
            try:
                self.sm.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                for n, bit in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(n)
            except Exception:
                pass
            self.stop.wait(0.005)

    def __enter__(self):
        try:
            nv, h = self._nvml_handle()
            self.mx = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            self.t = threading.Thread(target=self._poll_nvml, args=(nv, h), daemon=True)
            self.t.start()
            return self
        except Exception:
            pass
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read_smi, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read_smi(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                self.sm.append(float(parts[0]))
                self.mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(list(self.REASONS), parts[2:6]):
                if v.lower().startswith("active"):
                    self.reasons.add(n)

    def __exit__(self, *a):
        self.stop.set()
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.t:
            self.t.join(timeout=2)

    def summary(self):
        loaded = [s for s in self.sm if self.mx and s > 0.5 * self.mx] or self.sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": self.mx,
                "reasons": sorted(self.reasons), "samples": len(self.sm)}


# ------------------------------------------------------------- distributed
def dist_setup():
    import torch
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    return ws, rank, local


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(v, ws):
    if ws == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# -------------------------------------------------------------- CPU legs
def cpu_reference_sht(nfields_per_thread=2, threads=None):
    """Reference CPU SHT round trip at 721x1440 on the host cores (bounded sample)."""
    import oracle
    threads = threads or os.cpu_count() or 1
    n = threads * nfields_per_thread
    x = oracle.random_field((n, NLAT, NLON), 1)
    if oracle.ref_available():
        steady, tables, _ = oracle.ref().bench_sht_roundtrip(0, NLAT, NLON, LMAX, MMAX, x, threads)
        kind = "reference"
    else:  # C restatement, one field per task
        from concurrent.futures import ThreadPoolExecutor
        o = oracle.orc()
        t0 = time.perf_counter()

        def one(i):
            c = o.sht_forward(0, NLAT, NLON, LMAX, MMAX, x[i:i + 1])
            o.sht_inverse(0, NLAT, NLON, c)
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(one, range(n)))
        steady, tables, kind = time.perf_counter() - t0, 0.0, "port"
    return {"value": n / steady, "unit": UNIT, "cores": threads, "kind": kind,
            "sample": f"{n} fields of 721x1440 equiangular, SHT+ISHT round trip (lmax=721, mmax=720), "
                      f"{threads} threads x {nfields_per_thread} fields; one-time Legendre tables "
                      f"{tables:.1f} s excluded", "seconds": steady, "tables_s": tables}


def cpu_reference_disco(threads=None):
    """Reference disco_apply at configs[2] for ONE sample (64 -> 256 channels), measured on
    a 16-input-channel slice with all 256 outputs and scaled by 64/16: both terms of the
    reference's cost -- the gather (convolution.hpp:192-205) and the mix (:207-218) -- are
    linear in c_in, so the scaling is exact (the former 8-output sample under-counted the
    c_out-proportional mix)."""
    import oracle
    threads = threads or os.cpu_count() or 1
    cin_s, cin, cout = 16, 64, 256
    x = oracle.random_field((cin_s, NLAT, NLON), 1)
    mix = oracle.random_field((cout, cin_s, 9), 77)
    steady, asm, _ = oracle.ref().bench_disco(0, NLAT, NLON, 1, 360, 720, 3 * math.pi / 360, x,
                                              mix, min(threads, cin_s))
    t_sample = steady * cin / cin_s
    return {"value": cout / t_sample, "unit": "output fields/s", "cores": min(threads, cin_s), "kind": "reference",
            "sample": f"DISCO 721x1440->360x720, c_in 16 of 64 with all 256 outputs on {min(threads, cin_s)} "
                      f"threads (reference threads over c_in), time x 64/16 (gather and mix are linear in "
                      f"c_in); assembly {asm:.1f} s excluded", "seconds": t_sample}


def run_reference_arm(args, ws, rank):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    vals = []
    info = None
    for i in range(args.warmup + args.steps):
        info = cpu_reference_disco(threads) if args.workload == "disco" else cpu_reference_sht(1, threads)
        if i >= args.warmup:
            vals.append(info["value"])
    v = statistics.median(vals)
    out = {"metric": METRIC, "value": v, "unit": info["unit"], "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * info["seconds"],
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (oracles.hpp random_field stream)", "impl": "reference",
           "config": workload_config(args),
           "cpu_baseline": {k: info[k] for k in ("value", "unit", "cores", "kind", "sample")},
           "e2e": {"value": v, "unit": info["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


SHT_CONFIG = {"workload": "configs[1]: forward+inverse SHT, 721x1440 equiangular (lmax=720 i.e. reference counts "
                          "lmax=721, mmax=720), 256 channels x batch 4 per GPU",
              "grid": "equiangular 721x1440", "fields_per_gpu": FIELDS, "batch": BATCH, "channels": CHANNELS,
              "precision": "fp32 I/O, 3xTF32 tcgen05 Legendre GEMMs, fp32 accumulate",
              "l2_policy": "inputs (4.25 GB/GPU) larger than the 126 MB L2"}
DISCO_CONFIG = {"workload": "configs[2]: DISCO conv 721x1440 eq -> 360x720 Gaussian, Morlet K=9, cutoff 3pi/360, "
                            "64 -> 256 channels, batch 4 per GPU",
                "batch": 4, "c_in": 64, "c_out": 256, "precision": "fp32 I/O, 3xTF32 channel mix",
                "l2_policy": "inputs (1.06 GB/GPU) larger than the 126 MB L2"}


def workload_config(args):
    if args.workload in ("all", "sht"):
        cfg = dict(SHT_CONFIG, parallelism=f"fields sharded over {args.gpus} GPU(s)")
        if args.workload == "all":
            cfg["also"] = ("cfg1: configs[0] (CUDA graph); disco: configs[2]; block: configs[3]; "
                           "domain_decomposed (N>1): configs[4]")
        return cfg
    if args.workload in ("dist_sht", "dist_disco"):
        nh, nw = decomp(args)
        what = ("forward + inverse SHT round trip (paper Alg. 1 and its mirror)" if args.workload == "dist_sht"
                else "DISCO conv -> 360x720 Gaussian, 512 -> 512 channels (Alg. 2 with latitude halo)")
        return {"workload": f"configs[4]: distributed {what}, 721x1440 equiangular, 512 channels, "
                            f"batch 1, {nh}x{nw} (polar x azimuth) decomposition",
                "decomposition": f"{nh}x{nw}", "channels": 512,
                "parallelism": f"lat/lon domain decomposition over {nh * nw} GPU(s), NCCL (libsphgpu.so)",
                "precision": "fp32 I/O, 3xTF32 tcgen05 GEMMs"}
    if args.workload == "block":
        return {"workload": "configs[3]: one global block (SHT -> spectral channel mix -> ISHT -> GeLU/MLP "
                            "epilogue) + one local block (DISCO 360x720 -> 360x720, Morlet K=9 -> MLP epilogue) "
                            "at 360x720 Gaussian, 256 channels, MLP hidden 512, batch 1",
                "batch": 1, "channels": 256, "mlp_hidden": 512, "precision": "fp32 I/O, 3xTF32 GEMMs"}
    if args.workload == "decoder":
        return {"workload": "§8f decoder group (model.hpp:372-394): bilinear upsample 360x720 Gaussian -> "
                            "721x1440 eq fused into DISCO 721x1440 -> 721x1440 (Morlet K=9, cutoff 3pi/720), "
                            "64 -> 64 channels, batch 4 per GPU",
                "batch": 4, "c_in": 64, "c_out": 64, "precision": "fp32 I/O, 3xTF32 channel mix"}
    if args.workload == "disco_t":
        return {"workload": "configs[2] adjoint: disco_transpose_apply 360x720 Gaussian -> 721x1440 eq, "
                            "Morlet K=9, cutoff 3pi/360, 256 -> 64 channels, batch 4 per GPU",
                "batch": 4, "c_in": 64, "c_out": 256, "precision": "fp32 I/O, 3xTF32 channel mix"}
    return dict(DISCO_CONFIG)


def decomp(args):
    ws = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    if args.decomp:
        nh, nw = (int(v) for v in args.decomp.lower().split("x"))
    else:
        nh, nw = ws, 1
    if nh * nw != ws:
        raise SystemExit(f"--decomp {nh}x{nw} does not match WORLD_SIZE={ws}")
    return nh, nw


# ----------------------------------------------------------------- timing
def timed(step, steps, warmup, ws, local, stream):
    """W warm-up steps, then K steps bracketed by barrier + synchronize, CUDA events on
    the launching stream, clocks sampled during the region; returns (ms/step max over
    ranks, library launches in the region, per-kernel profile, clock summary)."""
    import torch
    from paper_2507_12144_b200 import _lib as L
    for _ in range(max(warmup, 3)):
        step()
    torch.cuda.synchronize()
    L.profile_read()
    L.profile_enable(True)
    launches0 = L.launch_count()
    barrier(ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    barrier(ws)
    L.profile_enable(False)
    launches = L.launch_count() - launches0
    prof = L.profile_read()
    ms = max_over_ranks(e0.elapsed_time(e1) / steps, ws)
    return ms, launches, prof, clk.summary()


def roofline(prof, steps, ms, traffic_key=None):
    """Dominant kernel of the step from live CUDA-event timing of every library launch:
    GEMMs against the 3xTF32 tensor ceiling (measured bf16 / 2 for TF32, / 3 passes) on
    algorithmic 2MNK flops; everything else against measured HBM bandwidth on
    algorithmic bytes."""
    hbm, bf16, _, peak_src = peaks()
    if not prof:
        return None
    name, (cnt, tot_ms, work) = max(prof.items(), key=lambda kv: kv[1][1])
    per_launch_s = tot_ms / cnt / 1e3
    if name.startswith("gemm"):
        achieved = work / cnt / per_launch_s / 1e12
        pk = bf16 / 2 / 3
        roof = {"kernel": name, "bound": "tensor", "achieved": achieved, "peak": pk, "unit": "TFLOP/s",
                "frac": achieved / pk,
                "peak_note": f"{peak_src} bf16 {bf16} TF/s / 2 (TF32 rate) / 3 (3xTF32 passes)"}
    else:
        achieved = work / cnt / per_launch_s / 1e9
        roof = {"kernel": name, "bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "peak_note": f"{peak_src} copy bandwidth"}
    roof["share_of_step"] = tot_ms / steps / ms
    roof["algorithmic_per_launch"] = work / cnt
    roof["traffic"] = None
    try:  # DRAM bytes per launch of this kernel from the committed ncu capture
        with open(os.path.join(ROOT, "profiles", "ncu_traffic_sht.json")) as f:
            tj = json.load(f)
        tw = tj["dram_bytes_per_launch"] if traffic_key == "sht" else \
            tj.get("by_workload", {}).get(traffic_key, {}).get("dram_bytes_per_launch", {})
        if name in tw:
            roof["traffic"] = tw[name]
            roof["traffic_unit"] = "bytes/launch (ncu dram__bytes_read+write)"
    except Exception:
        pass
    roof["per_kernel_ms"] = {k: v[1] / steps for k, v in sorted(prof.items())}
    # every kernel of the step against its own bound (north_star: tensor-pipe fraction for
    # the GEMMs, HBM fraction for the FFT / DISCO kernels), from the same live timings
    per = {}
    for k, (n, t_ms, w) in sorted(prof.items()):
        if n == 0 or t_ms <= 0 or w <= 0:
            continue
        if k.startswith("gemm"):
            a = w / (t_ms / 1e3) / 1e12
            per[k] = {"bound": "tensor", "achieved_TFLOPs": a, "frac": a / (bf16 / 2 / 3)}
        else:
            a = w / (t_ms / 1e3) / 1e9
            per[k] = {"bound": "hbm", "achieved_GBps": a, "frac": a / hbm}
    roof["per_kernel"] = per
    try:  # ncu counters of the same kernels (committed capture, profiles/capture_r2.sh)
        with open(os.path.join(ROOT, "profiles", "ncu_traffic_sht.json")) as f:
            roof["ncu_tensor_pipe_active_pct"] = json.load(f).get("tensor_pipe_active_pct")
    except Exception:
        pass
    return roof


# ----------------------------------------------------------------- GPU arm
def measure_sht(args, ws, rank, local):
    import torch
    import paper_2507_12144_b200 as S
    from paper_2507_12144_b200 import _lib as L
    dev = torch.device("cuda", local)
    g = S.build_equiangular(NLAT, NLON)
    plan = S.ShtPlan(g, LMAX, MMAX, "3xtf32", allow_equiangular_forward=True, device=dev)
    F = FIELDS
    x = torch.rand((F, NLAT, NLON), device=dev, dtype=torch.float32) * 2 - 1
    y = torch.empty_like(x)
    cint = torch.zeros(plan.coeffs_elems(F, L.SPH_LAYOUT_INTERNAL), device=dev)
    wsb = plan.workspace(F)

    def step():
        plan.forward(x, L.SPH_LAYOUT_INTERNAL, out=cint, ws=wsb)
        plan.inverse(cint, F, L.SPH_LAYOUT_INTERNAL, out=y, ws=wsb)
    ms, launches, prof, clk = timed(step, args.steps, args.warmup, ws, local, torch.cuda.current_stream(dev))
    rec = {"value": ws * F / (ms / 1e3), "ms_per_step": ms, "gpu_launches": launches, "clocks": clk,
           "roofline": roofline(prof, args.steps, ms, "sht")}
    e2e = None
    if not args.no_e2e:  # end to end through the public C ABI with pinned host buffers
        xh = torch.empty((F, NLAT, NLON), dtype=torch.float32, pin_memory=True)
        xh.copy_(x)
        yh = torch.empty_like(xh, pin_memory=True)
        plan.roundtrip_host(xh, yh, chunk=args.chunk)  # warm-up (allocations, streams)
        barrier(ws)
        t0 = time.perf_counter()
        n_e2e = max(1, min(args.steps, 3))
        for _ in range(n_e2e):
            plan.roundtrip_host(xh, yh, chunk=args.chunk)
        t = max_over_ranks((time.perf_counter() - t0) / n_e2e, ws)
        e2e = {"value": ws * F / t, "unit": UNIT, "h2d_bytes_per_step": F * NLAT * NLON * 4,
               "d2h_bytes_per_step": F * NLAT * NLON * 4, "ms_per_step": t * 1e3,
               "api": "sph_sht_roundtrip_host (pinned host in/out; H2D, compute and D2H streams over 3 chunk "
                      "buffers)", "chunk_fields": args.chunk}
        del xh, yh
    rec["e2e"] = e2e
    # the same round trip through the REFERENCE coefficient layout ([F][lmax][mmax]
    # complex64, zeros above the diagonal) -- what a drop-in caller of sht_forward /
    # sht_inverse pays: the GEMM-native layout's conversions included
    del cint
    dense = torch.empty((F, LMAX, MMAX, 2), device=dev)

    def step_dense():
        plan.forward(x, L.SPH_LAYOUT_DENSE_LM, out=dense, ws=wsb)
        plan.inverse(dense, F, L.SPH_LAYOUT_DENSE_LM, out=y, ws=wsb)
    ms_d, launches_d, prof_d, _ = timed(step_dense, max(5, args.steps // 2), args.warmup, ws, local,
                                        torch.cuda.current_stream(dev))
    rec["reference_layout"] = {"value": ws * F / (ms_d / 1e3), "unit": UNIT, "ms_per_step": ms_d,
                               "gpu_launches": launches_d,
                               "per_kernel_ms": {k: v[1] / max(5, args.steps // 2) for k, v in sorted(prof_d.items())},
                               "api": "sph_sht_forward / sph_sht_inverse with SPH_LAYOUT_DENSE_LM"}
    del x, y, dense, wsb
    return rec


def measure_disco(args, ws, rank, local):
    import torch
    import paper_2507_12144_b200 as S
    dev = torch.device("cuda", local)
    hbm = peaks()[0]
    op = S.DiscoOperator(S.build_equiangular(NLAT, NLON), S.build_gaussian(360, 720),
                         S.morlet_basis(3 * math.pi / 360), device=dev)
    B, cin, cout = 4, 64, 256
    mix = (torch.rand((cout, cin, op.n_basis), device=dev) * 2 - 1) / math.sqrt(cin * 9)
    x = torch.rand((B, cin, NLAT, NLON), device=dev) * 2 - 1
    y = torch.empty((B, cout, 360, 720), device=dev)
    wsb = op.workspace(B, cin, cout)

    def step():
        op.apply(x, mix, out=y, ws=wsb)
    ms, launches, prof, clk = timed(step, args.steps, args.warmup, ws, local, torch.cuda.current_stream(dev))
    units = B * cout
    # SURVEY §8(d) compulsory bytes per step: x + y + psi (fp32 value + 2 indices per entry
    # and basis) + W
    comp = 4 * B * cin * NLAT * NLON + 4 * B * cout * 360 * 720 + op.nnz_per_basis * op.n_basis * 12 \
        + 4 * cout * cin * 9
    rec = {"value": ws * units / (ms / 1e3), "unit": "output fields/s", "ms_per_step": ms, "gpu_launches": launches,
           "clocks": clk, "config": dict(DISCO_CONFIG),
           "roofline": roofline(prof, args.steps, ms, "disco"),
           "step_hbm": {"compulsory_bytes": comp, "achieved_GBps": comp / (ms / 1e3) / 1e9, "peak": hbm,
                        "frac": comp / (ms / 1e3) / 1e9 / hbm,
                        "note": "SURVEY §8(d) compulsory bytes (x + y + psi + W) over the whole step time"}}
    e2e = None
    if not args.no_e2e:
        # per batch item: pinned host -> device (H2D stream), sph_disco_apply (compute
        # stream), device -> pinned host (D2H stream), 3 slots in flight
        xh = torch.empty((B, cin, NLAT, NLON), dtype=torch.float32, pin_memory=True)
        xh.copy_(x)
        yh = torch.empty((B, cout, 360, 720), dtype=torch.float32, pin_memory=True)
        NS = 3
        xd = [torch.empty((1, cin, NLAT, NLON), device=dev) for _ in range(NS)]
        yd = [torch.empty((1, cout, 360, 720), device=dev) for _ in range(NS)]
        ws1 = op.workspace(1, cin, cout)
        s_up, s_cp, s_dn = (torch.cuda.Stream(dev) for _ in range(3))
        ev_up = [torch.cuda.Event() for _ in range(NS)]
        ev_cp = [torch.cuda.Event() for _ in range(NS)]
        ev_dn = [torch.cuda.Event() for _ in range(NS)]

        def e2e_step():
            for b in range(B):
                k = b % NS
                with torch.cuda.stream(s_up):
                    s_up.wait_event(ev_cp[k])          # slot's input consumed
                    xd[k].copy_(xh[b:b + 1], non_blocking=True)
                    ev_up[k].record(s_up)
                with torch.cuda.stream(s_cp):
                    s_cp.wait_event(ev_up[k])
                    s_cp.wait_event(ev_dn[k])          # slot's output downloaded
                    op.apply(xd[k], mix, out=yd[k], ws=ws1)
                    ev_cp[k].record(s_cp)
                with torch.cuda.stream(s_dn):
                    s_dn.wait_event(ev_cp[k])
                    yh[b:b + 1].copy_(yd[k], non_blocking=True)
                    ev_dn[k].record(s_dn)
            torch.cuda.synchronize()
        e2e_step()
        barrier(ws)
        t0 = time.perf_counter()
        n_e2e = max(1, min(args.steps, 3))
        for _ in range(n_e2e):
            e2e_step()
        t = max_over_ranks((time.perf_counter() - t0) / n_e2e, ws)
        e2e = {"value": ws * units / t, "unit": "output fields/s", "h2d_bytes_per_step": xh.numel() * 4,
               "d2h_bytes_per_step": yh.numel() * 4, "ms_per_step": t * 1e3,
               "api": "sph_disco_apply per batch item (pinned host in/out; H2D, compute and D2H streams, 3 slots)"}
        del xh, yh, xd, yd, ws1
    rec["e2e"] = e2e
    del x, y, wsb
    # the adjoint on the same operator (disco_transpose_apply, convolution.hpp:226-266; the
    # DISCO backward pass w.r.t. its input): 256 -> 64 channels back onto 721x1440
    from paper_2507_12144_b200 import _lib as L
    v = torch.rand((B, cout, 360, 720), device=dev) * 2 - 1
    yt = torch.empty((B, cin, NLAT, NLON), device=dev)
    wst = torch.empty(L.lib.sph_disco_transpose_workspace_bytes(op.h, B, cin, cout), dtype=torch.uint8, device=dev)
    ms_t, launches_t, prof_t, _ = timed(lambda: op.transpose_apply(v, mix, out=yt, ws=wst), max(5, args.steps // 2),
                                        args.warmup, ws, local, torch.cuda.current_stream(dev))
    rec["transpose"] = {"workload": "disco_transpose_apply 360x720 -> 721x1440, 256 -> 64 channels, batch 4",
                        "value": ws * B * cin / (ms_t / 1e3), "unit": "output fields/s", "ms_per_step": ms_t,
                        "gpu_launches": launches_t,
                        "per_kernel_ms": {k: w[1] / max(5, args.steps // 2) for k, w in sorted(prof_t.items())}}
    del v, yt, wst
    return rec


def measure_cfg1(args, ws, rank, local):
    """configs[0]: SHT -> ISHT round trip, 91x180 equiangular (lmax 91 / mmax 90), 32
    fields -- latency-bound, so it runs as ONE CUDA-graph launch (the library's calls are
    stream-ordered and capture); the eager time is reported beside it."""
    import torch
    import paper_2507_12144_b200 as S
    from paper_2507_12144_b200 import _lib as L
    dev = torch.device("cuda", local)
    p = S.ShtPlan(S.build_equiangular(91, 180), 91, 90, "3xtf32", allow_equiangular_forward=True, device=dev)
    F = 32
    x = torch.rand((F, 91, 180), device=dev) * 2 - 1
    c = torch.zeros(p.coeffs_elems(F, L.SPH_LAYOUT_INTERNAL), device=dev)
    y = torch.empty_like(x)
    wsb = p.workspace(F)
    s = torch.cuda.Stream(dev)

    def step():
        p.forward(x, L.SPH_LAYOUT_INTERNAL, out=c, ws=wsb)
        p.inverse(c, F, L.SPH_LAYOUT_INTERNAL, out=y, ws=wsb)
    with torch.cuda.stream(s):
        eager_ms, _, _, _ = timed(step, 50, 5, ws, local, s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            step()
        graph_ms, launches, _, clk = timed(g.replay, 50, 5, ws, local, s)
    return {"workload": "configs[0]: SHT->ISHT round trip, 91x180 equiangular (lmax=91, mmax=90), 32 fields",
            "value": ws * F / (graph_ms / 1e3), "unit": "fields/s", "ms_per_step": graph_ms,
            "eager_ms_per_step": eager_ms, "launch": "one CUDA graph replay per step (4 library kernels)",
            "clocks": clk}


def measure_block(args, ws, rank, local):
    """configs[3]: one global block (SHT -> spectral channel mix -> ISHT -> GeLU/MLP
    epilogue) + one local block (DISCO 360x720 -> 360x720 -> MLP epilogue), 256 channels,
    MLP hidden 512, batch 1."""
    import torch
    import paper_2507_12144_b200 as S
    dev = torch.device("cuda", local)
    g = S.build_gaussian(360, 720)
    C, H, B = 256, 512, 1
    lat = S.SphericalField(g, torch.rand((B, C, 360, 720), device=dev) * 2 - 1)
    cond = S.SphericalField(g, torch.empty((B, 0, 360, 720), device=dev))
    sc = 1.0 / math.sqrt(C)

    def wts(conv):
        return S.BlockWeights(global_=conv.shape[2] != 9, conv=conv,
                              w1=(torch.rand((H, C), device=dev) * 2 - 1) * sc,
                              b1=torch.rand(H, device=dev) * 0.1,
                              w2=(torch.rand((C, H), device=dev) * 2 - 1) / math.sqrt(H),
                              b2=torch.rand(C, device=dev) * 0.1, scales=torch.full((C,), 0.1, device=dev))
    bw_g = wts((torch.rand((C, C, 360), device=dev) * 2 - 1) * sc)
    block_op = S.DiscoOperator(g, g, S.morlet_basis(3 * math.pi / 360), device=dev)
    bw_l = wts((torch.rand((C, C, block_op.n_basis), device=dev) * 2 - 1) * sc / 3)

    def step():
        S.block_apply(lat, cond, bw_g)
        S.block_apply(lat, cond, bw_l, block_op)
    ms, launches, prof, clk = timed(step, max(5, args.steps // 2), args.warmup, ws, local,
                                    torch.cuda.current_stream(dev))
    return {"workload": "configs[3]: global + local block pair at 360x720 Gaussian, 256 channels, MLP hidden 512, "
                        "batch 1", "value": ws * B * C / (ms / 1e3), "unit": "fields/s (block-pair outputs)",
            "ms_per_step": ms, "gpu_launches": launches, "clocks": clk,
            "per_kernel_ms": {k: v[1] / max(5, args.steps // 2) for k, v in sorted(prof.items())}}


def measure_domain_decomposed(args, ws, rank, local, nh, nw, steps):
    """configs[4] through the library's NCCL path: distributed SHT + inverse SHT round trip
    and distributed DISCO (721x1440 -> 360x720 Gaussian), 512 channels, batch 1.  The same
    problem on ONE GPU (rank 0 alone, the single-GPU plans) gives T1 for the strong-scaling
    efficiency T1 / (N * T_N)."""
    import torch
    import torch.distributed as dist
    import paper_2507_12144_b200 as S
    from paper_2507_12144_b200 import _lib as L
    from paper_2507_12144_b200 import dist as D
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    if not dist.is_initialized():  # one rank: a 1-process group carries the NCCL id
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29517")
        dist.init_process_group("nccl", device_id=dev, rank=0, world_size=1)
    C = 512
    grid = S.build_equiangular(NLAT, NLON)
    gout = S.build_gaussian(360, 720)
    op = S.DiscoOperator(grid, gout, S.morlet_basis(3 * math.pi / 360), device=dev)
    torch.manual_seed(99)
    mix = ((torch.rand((C, C, op.n_basis)) * 2 - 1) / math.sqrt(C * 9)).to(dev)
    out = {"decomposition": f"{nh}x{nw}", "channels": C, "batch": 1, "scaling": "strong",
           "api": "sph_dist_sht_forward / sph_dist_sht_inverse / sph_dist_disco_apply (NCCL, libsphgpu.so)"}

    def ev_time(step, n):
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(n):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / n

    # T1: rank 0 alone, single-GPU plans on the whole problem
    t1 = {}
    if rank == 0:
        p1 = S.get_sht_plan(grid, LMAX, MMAX, "3xtf32", allow_equiangular_forward=True, device=dev)
        xg = torch.rand((C, NLAT, NLON), device=dev) * 2 - 1
        cg = torch.empty((C, LMAX, MMAX, 2), device=dev)
        yg = torch.empty_like(xg)
        wsg = p1.workspace(C)

        def rt1():
            p1.forward(xg, L.SPH_LAYOUT_DENSE_LM, out=cg, ws=wsg)
            p1.inverse(cg, C, L.SPH_LAYOUT_DENSE_LM, out=yg, ws=wsg)
        t1["sht_roundtrip"] = ev_time(rt1, steps)
        yd = torch.empty((1, C, 360, 720), device=dev)
        wsd = op.workspace(1, C, C)
        t1["disco"] = ev_time(lambda: op.apply(xg[None], mix, out=yd, ws=wsd), steps)
        del xg, cg, yg, wsg, yd, wsd
        torch.cuda.empty_cache()
    dist.barrier()
    comm = D.NcclComm(D.CommGrid((1, 1, nh, nw)), device=dev)
    sp = D.DistShtPlan(comm, grid, LMAX, MMAX, C)
    dp = D.DistDiscoPlan(comm, op, C, C)
    x = torch.rand((C, sp.hn, sp.wn), device=dev) * 2 - 1
    c = torch.empty((C, sp.ln, sp.mn, 2), device=dev)
    y = torch.empty_like(x)
    xd = torch.rand((C, dp.hn, dp.wn), device=dev) * 2 - 1
    yd = torch.empty((C, dp.hon, dp.won), device=dev)

    def rt():
        sp.forward(x, out=c)
        sp.inverse(c, out=y)
    res = {}
    for name, step in (("sht_roundtrip", rt), ("disco", lambda: dp.apply(xd, mix, out=yd))):
        ms, launches, prof, clk = timed(step, steps, 3, ws, local, stream)
        r = {"ms_per_step": ms, "value": C / (ms / 1e3), "unit": "fields/s" if name != "disco" else "output fields/s",
             "gpu_launches": launches, "per_kernel_ms_rank0": {k: v[1] / steps for k, v in sorted(prof.items())}}
        if rank == 0:
            r["t1_ms"] = t1[name]
            r["strong_scaling_eff"] = t1[name] / (ws * ms)
        res[name] = r
    comm.traffic_reset()
    rt()
    dp.apply(xd, mix, out=yd)
    torch.cuda.synchronize()
    out.update(res)
    out["traffic_csv"] = comm.traffic_csv()
    del sp, dp
    comm.close()
    return out


def run_all(args, ws, rank, local):
    """The default line: configs[1] SHT (value), configs[2] DISCO, configs[4] (N > 1)."""
    sht = measure_sht(args, ws, rank, local)
    disco = measure_disco(args, ws, rank, local)
    cfg1 = measure_cfg1(args, ws, rank, local)
    block = measure_block(args, ws, rank, local)
    dd = measure_domain_decomposed(args, ws, rank, local, ws, 1, max(5, args.steps // 2)) if ws > 1 else None
    cpu = dcpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        try:
            cpu = {k: v for k, v in cpu_reference_sht(2).items() if k in ("value", "unit", "cores", "kind", "sample")}
        except Exception as ex:  # noqa: BLE001
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "unavailable", "sample": str(ex)}
        try:
            dcpu = {k: v for k, v in cpu_reference_disco().items()
                    if k in ("value", "unit", "cores", "kind", "sample")}
        except Exception as ex:  # noqa: BLE001
            dcpu = {"value": None, "unit": "output fields/s", "cores": 0, "kind": "unavailable", "sample": str(ex)}
    if rank == 0:
        disco["cpu_baseline"] = dcpu
        out = {"metric": METRIC, "value": sht["value"], "unit": UNIT, "n_gpus": ws, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": sht["ms_per_step"], "higher_is_better": True,
               "scaling": "weak", "vs_baseline": None, "dtype": "f32",
               "data": "synthetic (uniform(-1,1) fields of the named shape)", "config": workload_config(args),
               "roofline": sht["roofline"], "cpu_baseline": cpu, "e2e": sht["e2e"],
               "gpu_launches": sht["gpu_launches"], "clocks": sht["clocks"],
               "reference_layout": sht["reference_layout"], "disco": disco,
               "cfg1": cfg1, "block": block}
        if dd is not None:
            out["domain_decomposed"] = dd
        print(json.dumps(out), flush=True)


def run_ours(args, ws, rank, local):
    """Single-workload lines (development / profiling): sht, disco, disco_t, block, decoder."""
    import torch
    import paper_2507_12144_b200 as S
    from paper_2507_12144_b200 import _lib as L
    dev = torch.device("cuda", local)
    torch.manual_seed(1234 + rank)
    if args.workload in ("sht", "disco"):
        rec = (measure_sht if args.workload == "sht" else measure_disco)(args, ws, rank, local)
        cpu = None
        if rank == 0 and ws == 1 and not args.no_cpu:
            try:
                cpu = cpu_reference_sht(2) if args.workload == "sht" else cpu_reference_disco()
                cpu = {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")}
            except Exception as ex:  # noqa: BLE001
                cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "unavailable", "sample": str(ex)}
        if rank == 0:
            out = {"metric": METRIC, "value": rec["value"], "unit": rec.get("unit", UNIT), "n_gpus": ws,
                   "steps": args.steps, "warmup": args.warmup, "ms_per_step": rec["ms_per_step"],
                   "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
                   "data": "synthetic (uniform(-1,1) fields of the named shape)", "config": workload_config(args),
                   "roofline": rec["roofline"], "cpu_baseline": cpu, "e2e": rec["e2e"],
                   "gpu_launches": rec["gpu_launches"], "clocks": rec["clocks"]}
            for k in ("step_hbm", "reference_layout"):
                if k in rec:
                    out[k] = rec[k]
            print(json.dumps(out), flush=True)
        return
    extra = {}
    if args.workload == "block":
        g = S.build_gaussian(360, 720)
        C, H, B = 256, 512, 1
        lat = S.SphericalField(g, torch.rand((B, C, 360, 720), device=dev) * 2 - 1)
        cond = S.SphericalField(g, torch.empty((B, 0, 360, 720), device=dev))
        sc = 1.0 / math.sqrt(C)

        def wts(conv):
            return S.BlockWeights(global_=conv.shape[2] != 9, conv=conv,
                                  w1=(torch.rand((H, C), device=dev) * 2 - 1) * sc,
                                  b1=torch.rand(H, device=dev) * 0.1,
                                  w2=(torch.rand((C, H), device=dev) * 2 - 1) / math.sqrt(H),
                                  b2=torch.rand(C, device=dev) * 0.1, scales=torch.full((C,), 0.1, device=dev))
        bw_g = wts((torch.rand((C, C, 360), device=dev) * 2 - 1) * sc)
        block_op = S.DiscoOperator(g, g, S.morlet_basis(3 * math.pi / 360), device=dev)
        bw_l = wts((torch.rand((C, C, block_op.n_basis), device=dev) * 2 - 1) * sc / 3)

        def step():
            S.block_apply(lat, cond, bw_g)
            S.block_apply(lat, cond, bw_l, block_op)
        units = B * C
    elif args.workload == "decoder":
        gl, go = S.build_gaussian(360, 720), S.build_equiangular(NLAT, NLON)
        op = S.DiscoOperator(go, go, S.morlet_basis(3 * math.pi / 720), device=dev)
        dplan = S.DecoderPlan(op, gl)
        B, cin, cout = 4, 64, 64
        mix = (torch.rand((cout, cin, op.n_basis), device=dev) * 2 - 1) / math.sqrt(cin * 9)
        lat = torch.rand((B, cin, 360, 720), device=dev) * 2 - 1
        y = torch.empty((B, cout, NLAT, NLON), device=dev)
        wsb = torch.empty(L.lib.sph_decoder_workspace_bytes(dplan.h, B, cin, cout), dtype=torch.uint8, device=dev)

        def step():
            dplan.apply(lat, mix, out=y, ws=wsb)
        units = B * cout
    else:  # disco_t: disco_transpose_apply, v on the 360x720 grid -> 721x1440 (64 channels)
        op = S.DiscoOperator(S.build_equiangular(NLAT, NLON), S.build_gaussian(360, 720),
                             S.morlet_basis(3 * math.pi / 360), device=dev)
        B, cin, cout = 4, 64, 256
        mix = (torch.rand((cout, cin, op.n_basis), device=dev) * 2 - 1) / math.sqrt(cin * 9)
        v = torch.rand((B, cout, 360, 720), device=dev) * 2 - 1
        y = torch.empty((B, cin, NLAT, NLON), device=dev)
        wsb = torch.empty(L.lib.sph_disco_transpose_workspace_bytes(op.h, B, cin, cout), dtype=torch.uint8,
                          device=dev)

        def step():
            op.transpose_apply(v, mix, out=y, ws=wsb)
        units = B * cin
    ms, launches, prof, clk = timed(step, args.steps, args.warmup, ws, local, torch.cuda.current_stream(dev))
    if rank == 0:
        out = {"metric": METRIC, "value": ws * units / (ms / 1e3), "unit": "output fields/s", "n_gpus": ws,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
               "scaling": "weak", "vs_baseline": None, "dtype": "f32",
               "data": "synthetic (uniform(-1,1) fields of the named shape)", "config": workload_config(args),
               "roofline": roofline(prof, args.steps, ms, args.workload), "cpu_baseline": None, "e2e": None,
               "gpu_launches": launches, "clocks": clk}
        out.update(extra)
        print(json.dumps(out), flush=True)


def run_dist(args, ws, rank, local):
    """configs[4] alone at an explicit decomposition (--decomp NHxNW)."""
    nh, nw = decomp(args)
    dd = measure_domain_decomposed(args, ws, rank, local, nh, nw, args.steps)
    if rank == 0:
        r = dd["sht_roundtrip" if args.workload == "dist_sht" else "disco"]
        out = {"metric": METRIC, "value": r["value"], "unit": r["unit"], "n_gpus": ws, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": r["ms_per_step"], "higher_is_better": True,
               "scaling": "strong", "vs_baseline": None, "dtype": "f32",
               "data": "synthetic (uniform(-1,1) fields of the named shape)", "config": workload_config(args),
               "roofline": None, "cpu_baseline": None, "e2e": None, "gpu_launches": r["gpu_launches"],
               "domain_decomposed": dd}
        print(json.dumps(out), flush=True)


def self_launch(args):
    """``python bench.py --gpus N`` outside torchrun: start the N ranks ourselves."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="all",
                    choices=["all", "sht", "disco", "disco_t", "block", "decoder", "dist_sht", "dist_disco"])
    ap.add_argument("--decomp", default="", help="dist_*: NHxNW polar x azimuth ranks (default WORLD_SIZE x 1)")
    ap.add_argument("--chunk", type=int, default=32)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    env_ws = os.environ.get("WORLD_SIZE")
    if env_ws is None and args.gpus > 1:
        sys.exit(self_launch(args))
    if env_ws is not None and int(env_ws) != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={env_ws}")
    if args.impl == "reference":
        run_reference_arm(args, int(env_ws or "1"), int(os.environ.get("RANK", "0")))
        return
    ws, rank, local = dist_setup()
    if args.workload.startswith("dist_"):
        run_dist(args, ws, rank, local)
    elif args.workload == "all":
        run_all(args, ws, rank, local)
    else:
        run_ours(args, ws, rank, local)
    import torch.distributed as dist
    if dist.is_initialized():
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
