import sys
sys.path.insert(0, "/root/repo")
import paper_1904_06971_b200 as pkg
from paper_1904_06971_b200 import _lib
for geom, p, sp, f in [("coons_quadratic", 2, (7, 9), "biharmonic"), ("coons_rational", 2, (7, 9), "biharmonic"),
                       ("coons_rational", 2, (9, 9), "biharmonic"), ("coons_rational", 2, (12, 12), "biharmonic"),
                       ("coons_rational", 2, (7, 9), "poisson"), ("coons_rational", 2, (7, 9), "mass"),
                       ("coons_rational", 3, (7, 9), "biharmonic"), ("coons_quadratic", 2, (12, 12), "biharmonic")]:
    disc = pkg.make_discretization(pkg.builtin_domain(geom), p, sp)
    try:
        A = pkg.assemble(pkg.FormKind(f), disc)
        print(geom, p, sp, f, "ok", _lib.last_kernel_times()[-1][0])
    except Exception as e:
        print(geom, p, sp, f, "ERR", str(e)[:80])
        break
