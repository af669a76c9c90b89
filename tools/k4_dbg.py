"""K4 timing experiments (results are NOT valid under SG_K4_DBG != 0): config-5 full assembly kernel time."""
import os
import subprocess
import sys

code = '''
import sys; sys.path.insert(0, ".")
import paper_1904_06971_b200 as pkg
from paper_1904_06971_b200 import _lib
from paper_1904_06971_b200.configs import CONFIGS
cfg = CONFIGS[5]
disc = pkg.make_discretization(cfg.geom(), cfg.p, cfg.spans)
for form in ("poisson", "mass"):
    best = 1e9
    for _ in range(3):
        res, _, _ = pkg.assemble_device(pkg.FormKind(form), disc)
        best = min(best, dict(_lib.last_kernel_times())["assemble_mma"])
        res.free()
    print(form, round(best, 3), flush=True)
'''
for dbg in sys.argv[1:]:
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=dict(os.environ, SG_K4_DBG=dbg))
    print("SG_K4_DBG", dbg, r.stdout.strip().replace("\n", " | ") or r.stderr[-300:], flush=True)
