"""cfg2 SHT round trip (1024 fields): forward-then-inverse vs the pipelined device round trip
(sph_sht_roundtrip) over chunk sizes and GEMM CTA caps; checks the results agree.

Record of a reverted experiment: ShtPlan.roundtrip / sph_sht_roundtrip
were removed after this measured slower than forward-then-inverse, so the script no
longer runs against the current library."""
import sys
import torch
import paper_2507_12144_b200 as S
from paper_2507_12144_b200 import _lib as L

dev = torch.device("cuda", 0)
g = S.build_equiangular(721, 1440)
plan = S.ShtPlan(g, 721, 720, "3xtf32", allow_equiangular_forward=True)
F = 1024
x = torch.rand((F, 721, 1440), device=dev) * 2 - 1
y0 = torch.empty_like(x)
y1 = torch.empty_like(x)
cint = torch.zeros(plan.coeffs_elems(F, L.SPH_LAYOUT_INTERNAL), device=dev)
ws = plan.workspace(F)


def base():
    plan.forward(x, L.SPH_LAYOUT_INTERNAL, out=cint, ws=ws)
    plan.inverse(cint, F, L.SPH_LAYOUT_INTERNAL, out=y0, ws=ws)


def t(fn, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


print("forward+inverse", round(t(base), 3), "ms")
chunks = [int(a) for a in sys.argv[1].split(",")] if len(sys.argv) > 1 else [128, 256]
caps = [int(a) for a in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0, 120, 100]
for ch in chunks:
    for cap in caps:
        ms = t(lambda: plan.roundtrip(x, out=y1, chunk=ch, gemm_ctas=cap))
        err = ((y1 - y0).norm() / y0.norm()).item()
        print(f"roundtrip chunk {ch} cap {cap}: {ms:.3f} ms  rel diff vs fwd+inv {err:.2e}")
