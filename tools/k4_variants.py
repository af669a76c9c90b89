"""Device time of the config-5 full assemblies (both forms) with experimental builds: python tools/k4_variants.py <dir>..."""
import subprocess
import sys

code = '''
import sys; sys.path.insert(0, sys.argv[1])
import paper_1904_06971_b200 as pkg
from paper_1904_06971_b200 import _lib
from paper_1904_06971_b200.configs import CONFIGS
cfg = CONFIGS[5]
disc = pkg.make_discretization(cfg.geom(), cfg.p, cfg.spans)
for form in sys.argv[2].split(","):
    best = 1e9
    for _ in range(3):
        res, _, _ = pkg.assemble_device(pkg.FormKind(form), disc)
        kt = dict(_lib.last_kernel_times())
        best = min(best, kt["assemble_mma"])
        res.free()
    print(sys.argv[1], form, round(best, 3), flush=True)
'''
forms = "poisson"
for root in sys.argv[1:]:
    if root.startswith("--forms="):
        forms = root.split("=", 1)[1]
        continue
    r = subprocess.run([sys.executable, "-c", code, root, forms], capture_output=True, text=True, timeout=300)
    print(r.stdout.strip() or r.stderr[-300:], flush=True)
