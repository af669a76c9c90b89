"""Development: locate pattern differences of the surrogate divergence against a golden."""
import sys

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import numpy as np
import scipy.sparse as sp

import paper_1904_06971_b200 as pkg
from test_gpu_divergence import stokes_from_golden
from test_oracle_divergence import load_div

case = sys.argv[1] if len(sys.argv) > 1 else "sdiv_coons_quad_p2"
meta, arr = load_div(case)
st = stokes_from_golden(meta, arr)
D, rep = pkg.build_surrogate_divergence(st, pkg.ConstantSampling(meta["M"]), q=meta["q"])
for c, Dc in enumerate(D):
    G = sp.csr_matrix((arr[f"data_{c}"], arr[f"indices_{c}"], arr[f"indptr_{c}"]), shape=Dc.mat.shape)
    A = Dc.mat
    if np.array_equal(A.indptr, G.indptr) and np.array_equal(A.indices, G.indices):
        print(c, "pattern equal")
        continue
    Ad = A.tocoo()
    Gd = G.tocoo()
    sa = set(zip(Ad.row.tolist(), Ad.col.tolist()))
    sg = set(zip(Gd.row.tolist(), Gd.col.tolist()))
    for (r, cc) in sorted(sg - sa)[:10]:
        print(c, "missing in ours", r, cc, "golden value", G[r, cc], "row max", abs(G[r]).max())
    for (r, cc) in sorted(sa - sg)[:10]:
        print(c, "extra in ours", r, cc, "our value", A[r, cc], "row max", abs(A[r]).max())
