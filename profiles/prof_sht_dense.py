"""Driver for ncu captures of the reference-layout SHT round trip at cfg2 (the C_int <->
dense [F][lmax][mmax] transposes sht_to_dense / sht_from_dense)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2507_12144_b200 as S
from paper_2507_12144_b200 import _lib as L

F = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
g = S.build_equiangular(721, 1440)
p = S.ShtPlan(g, 721, 720, "3xtf32", allow_equiangular_forward=True)
x = torch.rand((F, 721, 1440), device="cuda") * 2 - 1
y = torch.empty_like(x)
c = torch.zeros(p.coeffs_elems(F, L.SPH_LAYOUT_DENSE_LM), device="cuda")
ws = p.workspace(F)
for _ in range(reps):
    p.forward(x, L.SPH_LAYOUT_DENSE_LM, out=c, ws=ws)
    p.inverse(c, F, L.SPH_LAYOUT_DENSE_LM, out=y, ws=ws)
torch.cuda.synchronize()
print("ok")
