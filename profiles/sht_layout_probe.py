"""Time the single-GPU forward SHT at cfg5 size (512 fields, 721x1440) in the internal
vs the dense [F][lmax][mmax] layout and the 1x1 dist_sht_forward step, to locate the
non-kernel time of the distributed path."""
import torch
import paper_2507_12144_b200 as S
from paper_2507_12144_b200 import _lib as L

dev = torch.device("cuda", 0)
g = S.build_equiangular(721, 1440)
plan = S.ShtPlan(g, 721, 720, "3xtf32", allow_equiangular_forward=True)
F = 512
x = torch.rand((F, 721, 1440), device=dev)
ws = plan.workspace(F)
ci = torch.zeros(plan.coeffs_elems(F, L.SPH_LAYOUT_INTERNAL), device=dev)
cd = torch.empty((F, 721, 720, 2), device=dev)


def t(fn, n=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


print("fwd internal (prealloc)", t(lambda: plan.forward(x, L.SPH_LAYOUT_INTERNAL, out=ci, ws=ws)))
print("fwd dense (prealloc)", t(lambda: plan.forward(x, L.SPH_LAYOUT_DENSE_LM, out=cd, ws=ws)))
print("fwd dense (alloc)", t(lambda: plan.forward(x, L.SPH_LAYOUT_DENSE_LM)))
L.profile_read()
L.profile_enable(True)
plan.forward(x, L.SPH_LAYOUT_DENSE_LM, out=cd, ws=ws)
torch.cuda.synchronize()
L.profile_enable(False)
print({k: round(v[1], 3) for k, v in L.profile_read().items()})
