for d in . expbuild/g128 expbuild/g512; do python - $d <<'PY'
import sys
sys.path.insert(0, sys.argv[1])
import paper_1904_06971_b200 as pkg
from paper_1904_06971_b200 import _lib
from paper_1904_06971_b200.configs import CONFIGS
from paper_1904_06971_b200.surrogate import surrogate_device
out=[sys.argv[1]]
cfg = CONFIGS[5]
disc = pkg.make_discretization(cfg.geom(), cfg.p, cfg.spans)
for form in ("mass","poisson"):
  for path in ("full","surr"):
    best=1e9
    for _ in range(3):
        if path=="full": res,_,_ = pkg.assemble_device(pkg.FormKind(form), disc)
        else: res,_,_ = surrogate_device(pkg.FormKind(form), disc, cfg.M, 3, pkg.surrogate.DEFAULT_MODE[form].value)
        best=min(best, dict(_lib.last_kernel_times())["geom_D"]); res.free()
    out.append((form,path,round(best,3)))
print(out, flush=True)
PY
done
