# GEMM failure bisection over nlat (K = folded rows) for the Legendre GEMMs
for N in ${NLATS:-91 121 181 241 361 721}; do
python - <<PY 2>&1 | grep -v "^ \|^Trace\|^$" | tail -${TAILN:-2}
import sys, torch
sys.path.insert(0, ".")
import paper_2507_12144_b200 as S
from paper_2507_12144_b200 import _lib as L
n = $N
g = S.build_equiangular(n, 2 * (n - 1))
p = S.ShtPlan(g, n, n - 1, "3xtf32", allow_equiangular_forward=True)
x = torch.rand((64, n, 2 * (n - 1)), device="cuda")
c = p.forward(x, L.SPH_LAYOUT_INTERNAL)
torch.cuda.synchronize()
print("nlat", n, "ok")
PY
done
