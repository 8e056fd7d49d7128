"""Small library calls for compute-sanitizer (memcheck / racecheck / synccheck):
cfg1-sized SHT round trip (single-CTA and CTA-pair GEMM paths), DISCO forward + adjoint
(Fourier path and the fp32 direct anchor), spectral conv + block epilogue, decoder.
Run:  compute-sanitizer --tool <tool> python profiles/sanitize_cases.py"""
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_12144_b200 as S  # noqa: E402
from paper_2507_12144_b200 import _lib as L  # noqa: E402

dev = torch.device("cuda", 0)
torch.manual_seed(0)
PI = math.pi
g = S.build_equiangular(91, 180)
for F in (4, 65):  # 65 fields selects the cta_group::2 Legendre GEMM
    p = S.ShtPlan(g, 91, 90, "3xtf32", allow_equiangular_forward=True)
    x = torch.rand((F, 91, 180), device=dev) * 2 - 1
    c = p.forward(x)
    y = p.inverse(c, F)
    ci = p.forward(x, L.SPH_LAYOUT_INTERNAL)
    p.inverse(ci, F, L.SPH_LAYOUT_INTERNAL)
torch.cuda.synchronize()
gi, go = S.build_equiangular(91, 180), S.build_gaussian(45, 90)
for prec in ("3xtf32", "fp32"):
    op = S.DiscoOperator(gi, go, S.morlet_basis(3 * PI / 45), prec)
    u = torch.rand((2, 4, 91, 180), device=dev)
    mix = torch.rand((8, 4, 9), device=dev)
    v = op.apply(u, mix)
    op.transpose_apply(v, mix)
torch.cuda.synchronize()
gg = S.build_gaussian(45, 90)
x = S.SphericalField(gg, torch.rand((1, 16, 45, 90), device=dev))
S.spectral_conv(x, torch.rand((16, 16, 45), device=dev) * 0.1)
bw = S.BlockWeights(False, None, torch.rand((32, 16), device=dev), torch.rand(32, device=dev),
                    torch.rand((16, 32), device=dev), torch.rand(16, device=dev), torch.rand(16, device=dev))
S.block_epilogue(torch.rand((1, 16, 45, 90), device=dev), x.data, bw)
go2 = S.build_equiangular(17, 32)
dop = S.DiscoOperator(go2, go2, S.morlet_basis(3 * PI / 16))
S.decode_preclamp(dop, S.SphericalField(S.build_gaussian(8, 16), torch.rand((1, 3, 8, 16), device=dev)),
                  torch.rand((2, 3, 9), device=dev))
torch.cuda.synchronize()
print("sanitize cases done;", L.launch_count(), "library launches")
