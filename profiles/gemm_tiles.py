"""Per-tile k-block interval (cycles) by instruction-N band from an SPH_GEMM_TRACE tile dump."""
import sys
import numpy as np

for path in sys.argv[1:]:
    a = np.loadtxt(path, dtype=np.int64)
    n = int((a[:, 0] > 0).sum())
    t, info = a[:n, 0], a[:n, 1]
    ninst, nkb = info // 1000, info % 1000
    dt = np.diff(t)
    per = dt / nkb[:-1]
    out = [f"tiles {n} total {t[-1] - t[0]} cyc"]
    for lo, hi in [(160, 193), (96, 160), (48, 96), (0, 48)]:
        sel = (ninst[:-1] >= lo) & (ninst[:-1] < hi)
        if sel.any():
            out.append(f"N[{lo},{hi}) {np.median(per[sel]):5.0f}")
    print("  " + " | ".join(out))
