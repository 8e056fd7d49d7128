"""Ring FFT engines (four-step n = N1*45, Stockham 2/3/5-smooth, O(n^2) fallback)
against the oracle's rfft_bins (fft.hpp:97-104; test_fft.cpp:20-52 lengths)."""
import numpy as np
import pytest

from conftest import rel_l2

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle  # noqa: E402
import paper_2507_12144_b200 as S  # noqa: E402

DEV = torch.device("cuda", 0)


@pytest.mark.parametrize("n", [2, 4, 8, 12, 16, 20, 48, 64, 90, 128, 180, 360, 720, 1440, 14, 22, 33])
def test_fft_stage_vs_oracle(n):
    mmax = max(1, n // 2)
    g = S.build_equiangular(4, n)
    p = S.ShtPlan(g, mmax, mmax)
    rings = oracle.random_field((3, 5, n), 1000 + n)  # F=3 fields x 5 rings (odd ring count)
    out = p.fft_stage(torch.tensor(rings, dtype=torch.float32, device=DEV), 3, 5)
    torch.cuda.synchronize()
    o = out.cpu().numpy().astype(np.float64)
    got = o[..., 0] + 1j * o[..., 1]
    want = np.stack([oracle.orc().rfft_bins(r, mmax) for r in rings.reshape(-1, n)]).reshape(3, 5, mmax)
    want *= 2 * np.pi / n
    assert rel_l2(got, want) <= 2e-6, n
