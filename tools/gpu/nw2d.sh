for d in . expbuild/w12 expbuild/w20 expbuild/w24; do python - $d <<'PY'
import sys
sys.path.insert(0, sys.argv[1])
import paper_1904_06971_b200 as pkg
from paper_1904_06971_b200 import _lib
from paper_1904_06971_b200.configs import CONFIGS
out=[sys.argv[1]]
for ci in (2,4,1):
    cfg = CONFIGS[ci]
    disc = pkg.make_discretization(cfg.geom(), cfg.p, cfg.spans)
    for form in cfg.forms:
        best=1e9
        for _ in range(4):
            res,_,_ = pkg.assemble_device(pkg.FormKind(form), disc)
            best=min(best, dict(_lib.last_kernel_times())["assemble_mma"]); res.free()
        out.append((ci,form,round(best,3)))
print(out, flush=True)
PY
done
