"""Driver for ncu captures of DISCO at cfg3 (721x1440 eq -> 360x720 Gaussian, 64->256, B)."""
import math
import sys
import torch
sys.path.insert(0, ".")
import paper_2507_12144_b200 as S

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
op = S.DiscoOperator(S.build_equiangular(721, 1440), S.build_gaussian(360, 720), S.morlet_basis(3 * math.pi / 360))
x = torch.rand((B, 64, 721, 1440), device="cuda") * 2 - 1
mix = (torch.rand((256, 64, 9), device="cuda") * 2 - 1) / 24
y = torch.empty((B, 256, 360, 720), device="cuda")
ws = op.workspace(B, 64, 256)
for _ in range(reps):
    op.apply(x, mix, out=y, ws=ws)
torch.cuda.synchronize()
print("ok")
