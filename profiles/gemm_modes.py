"""Time the Legendre GEMMs alone in the three precision modes at cfg2 (F fields)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2507_12144_b200 as S
from paper_2507_12144_b200 import _lib as L

F = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
g = S.build_equiangular(721, 1440)
x = torch.rand((F, 721, 1440), device="cuda") * 2 - 1
for prec in ["3xtf32", "tf32"]:
    p = S.ShtPlan(g, 721, 720, prec, allow_equiangular_forward=True)
    c = torch.zeros(p.coeffs_elems(F, L.SPH_LAYOUT_INTERNAL), device="cuda")
    y = torch.empty_like(x)
    ws = p.workspace(F)
    for _ in range(3):
        p.forward(x, L.SPH_LAYOUT_INTERNAL, out=c, ws=ws)
        p.inverse(c, F, L.SPH_LAYOUT_INTERNAL, out=y, ws=ws)
    torch.cuda.synchronize()
    L.profile_read()
    L.profile_enable(True)
    for _ in range(10):
        p.forward(x, L.SPH_LAYOUT_INTERNAL, out=c, ws=ws)
        p.inverse(c, F, L.SPH_LAYOUT_INTERNAL, out=y, ws=ws)
    torch.cuda.synchronize()
    L.profile_enable(False)
    pr = L.profile_read()
    print(prec, {k: round(v[1] / v[0], 3) for k, v in pr.items()})
    del p, c, y, ws
    torch.cuda.empty_cache()
