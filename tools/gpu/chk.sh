bash tools/gpu/ms.sh 2>&1 | grep "^\["
python - <<'PY'
import sys
sys.path.insert(0, "expbuild/nc3")
import numpy as np
import paper_1904_06971_b200 as pkg
sys.path.insert(0, ".")
from oracle import surriga_oracle as O
disc3 = pkg.make_discretization(pkg.twisted_cube_standin(), 3, (14, 15, 13))
A3 = pkg.assemble(pkg.FormKind.POISSON, disc3)
ip, ix, d, _, _ = O.assemble(O.problem_from_disc(pkg.FormKind.POISSON, disc3))
m = A3.mat
print("nc3 parity", O.row_scaled_error(ip, ix, d, m.indptr.astype(np.int64), m.indices, m.data), pkg.is_bitwise_symmetric(A3))
PY
