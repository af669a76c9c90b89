"""clock64 breakdown of the warp-specialised K4 loop (experimental build, tools/expbuild.sh prof -DSG_K4_PROF):
python tools/k4_prof.py expbuild/prof [form]"""
import sys

sys.path.insert(0, sys.argv[1])
import paper_1904_06971_b200 as pkg  # noqa: E402
from paper_1904_06971_b200 import _lib  # noqa: E402
from paper_1904_06971_b200.configs import CONFIGS  # noqa: E402

cfg = CONFIGS[5]
disc = pkg.make_discretization(cfg.geom(), cfg.p, cfg.spans)
form = sys.argv[2] if len(sys.argv) > 2 else "poisson"
for _ in range(2):
    res, _, _ = pkg.assemble_device(pkg.FormKind(form), disc)
    print(form, dict(_lib.last_kernel_times())["assemble_mma"], flush=True)
    res.free()
