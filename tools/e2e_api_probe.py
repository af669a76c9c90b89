"""Wall time of each public-API call of the config-5 e2e step, split into device call, to_host and the
rest (scipy CSR + report): python tools/e2e_api_probe.py [steps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_06971_b200 as pkg  # noqa: E402
from paper_1904_06971_b200 import _lib  # noqa: E402
from paper_1904_06971_b200.configs import CONFIGS  # noqa: E402

cfg = CONFIGS[5]
disc = pkg.make_discretization(cfg.geom(), cfg.p, cfg.spans)
_lib.host_staging_init(0)
orig = _lib.Result.to_host
acc = {}


def timed_to_host(self):
    t = time.perf_counter()
    out = orig(self)
    acc["to_host"] = acc.get("to_host", 0.0) + time.perf_counter() - t
    return out


_lib.Result.to_host = timed_to_host
for step in range(int(sys.argv[1]) if len(sys.argv) > 1 else 5):
    row = []
    for f in cfg.forms:
        for path in ("full", "surrogate"):
            acc.clear()
            t0 = time.perf_counter()
            if path == "full":
                A = pkg.assemble(pkg.FormKind(f), disc)
            else:
                A, _ = pkg.build_surrogate_matrix(pkg.FormKind(f), disc, pkg.ConstantSampling(cfg.M), q=cfg.q)
            t1 = time.perf_counter()
            dev = _lib.last_timing()[0]
            row.append(f"{f[:4]}/{path[:4]} total {1e3 * (t1 - t0):6.1f} dev {dev:5.1f} to_host {1e3 * acc.get('to_host', 0):6.1f}")
            del A
    print(f"step {step}: " + " | ".join(row), flush=True)
    if step == 1:
        _lib.host_pool_sync()
