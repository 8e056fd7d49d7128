"""Where does the cfg4 local-block DISCO (360x720 Gaussian -> same, stride 1, Morlet
3pi/360, 256 -> 256) lose accuracy against the fp64 reference?  Compares the Fourier
3xTF32 path and the fp32 direct-gather anchor with the unmodified reference on output
channels {0, 128, 255}, and single-channel convolutions (mix one-hot per basis k)."""
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2507_12144_b200 as S  # noqa: E402

PI = math.pi
dev = torch.device("cuda", 0)
T = os.cpu_count()


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


g = S.build_gaussian(360, 720)
ops = {p: S.DiscoOperator(g, g, S.morlet_basis(3 * PI / 360), p) for p in ("3xtf32", "fp32")}
C = 256
x = oracle.random_field((C, 360, 720), 43)
mix = oracle.random_field((C, C, 9), 44) / 48.0
outs = [0, 128, 255]
_, _, ref = oracle.ref().bench_disco(1, 360, 720, 1, 360, 720, 3 * PI / 360, x, mix[outs], T, want_y=True)
for p, op in ops.items():
    y = op.apply(torch.tensor(x[None], dtype=torch.float32, device=dev),
                 torch.tensor(mix, dtype=torch.float32, device=dev))[0, outs].cpu().numpy().astype(np.float64)
    rows = [rel(y[:, h], ref[:, h]) for h in range(360)]
    print(p, "all", rel(y, ref), "worst rows", sorted(range(360), key=lambda h: -rows[h])[:6],
          [f"{rows[h]:.2e}" for h in sorted(range(360), key=lambda h: -rows[h])[:6]])
# single channel, one basis function at a time
x1 = x[:1]
for k in range(9):
    m1 = np.zeros((1, 1, 9))
    m1[0, 0, k] = 1.0
    _, _, r1 = oracle.ref().bench_disco(1, 360, 720, 1, 360, 720, 3 * PI / 360, x1, m1, 1, want_y=True)
    res = []
    for p, op in ops.items():
        y = op.apply(torch.tensor(x1[None], dtype=torch.float32, device=dev),
                     torch.tensor(m1, dtype=torch.float32, device=dev))[0].cpu().numpy().astype(np.float64)
        res.append(f"{p} {rel(y, r1):.2e}")
    print("k", k, *res, "norm", float(np.linalg.norm(r1)))
