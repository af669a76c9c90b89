for d in . expbuild/nb5 expbuild/nb6 expbuild/nb7; do python - $d <<'PY'
import sys
sys.path.insert(0, sys.argv[1])
import paper_1904_06971_b200 as pkg
from paper_1904_06971_b200 import _lib
from paper_1904_06971_b200.configs import CONFIGS
from paper_1904_06971_b200.surrogate import surrogate_device
out=[sys.argv[1]]
for ci in (3,5):
    cfg = CONFIGS[ci]
    disc = pkg.make_discretization(cfg.geom(), cfg.p, cfg.spans)
    for path in ("full","surr"):
        best=1e9
        for _ in range(3):
            if path=="full": res,_,_ = pkg.assemble_device(pkg.FormKind("poisson"), disc)
            else: res,_,_ = surrogate_device(pkg.FormKind("poisson"), disc, cfg.M, 3, pkg.surrogate.DEFAULT_MODE["poisson"].value)
            best=min(best, dict(_lib.last_kernel_times())["assemble_mma"]); res.free()
        out.append((ci,path,round(best,3)))
print(out, flush=True)
PY
done
