"""Reference-envelope probe: the oracle with pairwise (not OpenBLAS) dot products vs the
reference golden traces — how far the reference algorithm itself moves under a pure
reassociation.  Run: python tests/golden/envelope_probe.py"""
import sys, numpy as np
import os; ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))); sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle import blocksolve_oracle as O
from golden_io import arrays, meta
class PW(np.ndarray):
    def __matmul__(self, other): return np.add.reduce(np.asarray(self) * np.asarray(other))
orig = O.cg
def cg_pw(apply, b, x0, its, tol=0.0, basis="rhs"):
    ap = lambda v: apply(np.asarray(v)).view(PW)
    return orig(ap, np.asarray(b).view(PW), np.asarray(x0).view(PW), its, tol, basis)
O.cg = cg_pw
for key in ["outer/box_12_222", "outer/cfg3_16_paper", "outer/cfg1_16_fixed"]:
    A, M = arrays(), meta()[key]; c = M["case"]; n = c["n"]; kind, its, itol = c["inner"]
    r = O.outer_solve_sync((n,n,n), A[key+"/rhs"], tuple(c["bg"]), c["ov"], dict(kind=kind, max_iterations=its, tolerance=itol), tol=c["tol"], max_outer=c.get("max_outer",5000), residual_check_mode=c["mode"])
    ref = np.array([t[2] for t in M["trace"]]); mine = np.array([row.estimated_residual for row in r.rows])
    m = min(len(ref), len(mine))
    d = np.abs(ref[:m]-mine[:m]); rel = d/ref[:m]
    print(key, "outer", r.outer_iterations, M["outer_iterations"], "max abs", d.max(), "max rel", rel.max())
