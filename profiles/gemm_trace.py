"""Summarise SPH_GEMM_TRACE dumps (CTA 0 per-k-block clock64 stamps) from gemm_tc.cu."""
import sys
import numpy as np

for path in sys.argv[1:]:
    a = np.loadtxt(path, dtype=np.int64)
    j, p, l, c, m = a.T
    sl = slice(100, 480)
    print(path)
    print("  issue->land %6.0f  land->converted %6.0f  converted->mma %6.0f  mma(j)->issue(j+S) %6.0f  "
          "k-block interval %6.0f cyc" % (np.median((l - p)[sl]), np.median((c - l)[sl]), np.median((m - c)[sl]),
                                        np.median((p[4:] - m[:-4])[sl]), np.median(np.diff(m)[sl])))
