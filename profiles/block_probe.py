"""Host vs device time of the cfg4 block pair: CUDA-event step time against the sum of
the library's profiled kernels, with and without the Python-level concat."""
import math
import time
import torch
import paper_2507_12144_b200 as S
from paper_2507_12144_b200 import _lib as L

dev = torch.device("cuda", 0)
g = S.build_gaussian(360, 720)
C, H = 256, 512
lat = S.SphericalField(g, torch.rand((1, C, 360, 720), device=dev) * 2 - 1)
cond = S.SphericalField(g, torch.empty((1, 0, 360, 720), device=dev))
sc = 1.0 / math.sqrt(C)


def wts(conv):
    return S.BlockWeights(global_=conv.shape[2] != 9, conv=conv, w1=(torch.rand((H, C), device=dev) * 2 - 1) * sc,
                          b1=torch.rand(H, device=dev) * 0.1, w2=(torch.rand((C, H), device=dev) * 2 - 1) / math.sqrt(H),
                          b2=torch.rand(C, device=dev) * 0.1, scales=torch.full((C,), 0.1, device=dev))


bw_g = wts((torch.rand((C, C, 360), device=dev) * 2 - 1) * sc)
op = S.DiscoOperator(g, g, S.morlet_basis(3 * math.pi / 360))
bw_l = wts((torch.rand((C, C, op.n_basis), device=dev) * 2 - 1) * sc / 3)
for name, fn in [("global", lambda: S.block_apply(lat, cond, bw_g)), ("local", lambda: S.block_apply(lat, cond, bw_l, op))]:
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    L.profile_read()
    L.profile_enable(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(10):
        fn()
    e1.record()
    th = (time.perf_counter() - t0) / 10
    torch.cuda.synchronize()
    L.profile_enable(False)
    prof = L.profile_read()
    print(name, "device ms", round(e0.elapsed_time(e1) / 10, 3), "host issue ms", round(th * 1e3, 3),
          "profiled kernels ms", round(sum(v[1] for v in prof.values()) / 10, 3))
