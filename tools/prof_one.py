"""Run one assembly (for ncu): python tools/prof_one.py <geom> <p> <spans...> <form> [full|surrogate] [M]"""
import sys

sys.path.insert(0, ".")
import paper_1904_06971_b200 as pkg
from paper_1904_06971_b200 import _lib
from paper_1904_06971_b200.surrogate import surrogate_device

geom = {"twisted": pkg.twisted_cube_standin, "sinmap": pkg.sin_map_standin, "annulus": pkg.quarter_annulus}[sys.argv[1]]()
p = int(sys.argv[2])
form = None
spans = []
rest = sys.argv[3:]
while rest and rest[0].isdigit():
    spans.append(int(rest.pop(0)))
form = rest.pop(0)
path = rest.pop(0) if rest else "full"
M = int(rest.pop(0)) if rest else 16
disc = pkg.make_discretization(geom, p, tuple(spans))
for it in range(2):
    if path == "full":
        res, _, _ = pkg.assemble_device(pkg.FormKind(form), disc)
    else:
        res, _, _ = surrogate_device(pkg.FormKind(form), disc, M, 3, pkg.surrogate.DEFAULT_MODE[form].value)
    print(_lib.last_timing(), [(n, round(t, 3)) for n, t in _lib.last_kernel_times()], res.sizes(), flush=True)
    res.free()
