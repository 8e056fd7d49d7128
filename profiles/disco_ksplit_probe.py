"""cfg4 local DISCO (360x720 Gaussian, stride 1, 256 -> 256): relative error vs the fp64
reference as a function of how the c_in*K reduction of the 3xTF32 mix GEMM is split.
The split is emulated at the API level (apply per input-channel group, fp32 sum), which
is what a k-split GEMM with an fp32 (RNE) accumulate epilogue computes.  Also the BN=128
A_lo-in-TMEM kernel (cout <= 128) on the same reduction."""
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
g = S.build_gaussian(360, 720)
op = S.DiscoOperator(g, g, S.morlet_basis(3 * PI / 360))
C = 256
x = oracle.random_field((C, 360, 720), 43)
mix = oracle.random_field((C, C, 9), 44) / 48.0
outs = [0, 100, 128]
_, _, ref = oracle.ref().bench_disco(1, 360, 720, 1, 360, 720, 3 * PI / 360, x, mix[outs], os.cpu_count(),
                                     want_y=True)
xt = torch.tensor(x[None], dtype=torch.float32, device=dev)
mt = torch.tensor(mix, dtype=torch.float32, device=dev)


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


for cg in (256, 128, 64, 32, 16):
    y = torch.zeros((1, C, 360, 720), device=dev)
    for c0 in range(0, C, cg):
        y += op.apply(xt[:, c0:c0 + cg].contiguous(), mt[:, c0:c0 + cg].contiguous())
    print(f"BN256 k-split {cg} channels (K={cg * 9}): {rel(y[0, outs].cpu().numpy().astype(np.float64), ref):.3e}")
# BN = 128 A_lo-in-TMEM kernel (selected for cout <= 128): first 129 outputs in two halves
y = torch.cat([op.apply(xt, mt[:128].contiguous()), op.apply(xt, mt[128:].contiguous())], 1)
print(f"ALO BN128 full K=2304: {rel(y[0, outs].cpu().numpy().astype(np.float64), ref):.3e}")
y = torch.zeros((1, 128, 360, 720), device=dev)
for c0 in range(0, C, 64):
    y += op.apply(xt[:, c0:c0 + 64].contiguous(), mt[:128, c0:c0 + 64].contiguous())
print(f"ALO BN128 k-split 64 ch: {rel(y[0, [0, 100]].cpu().numpy().astype(np.float64), ref[:2]):.3e}")
