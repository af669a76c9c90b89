"""One full assembly per form at config 5 (for an ncu capture of each form's K4): python tools/prof_forms.py poisson mass"""
import sys

sys.path.insert(0, ".")
import paper_1904_06971_b200 as pkg  # noqa: E402
from paper_1904_06971_b200 import _lib  # noqa: E402
from paper_1904_06971_b200.configs import CONFIGS  # noqa: E402

cfg = CONFIGS[5]
disc = pkg.make_discretization(cfg.geom(), cfg.p, cfg.spans)
for form in sys.argv[1:]:
    res, _, _ = pkg.assemble_device(pkg.FormKind(form), disc)
    print(form, dict(_lib.last_kernel_times()), flush=True)
    res.free()
