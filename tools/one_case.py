import sys, numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
from golden_io import load
from gpu_util import disc_from_golden, form_of
import paper_1904_06971_b200 as pkg
from paper_1904_06971_b200 import _lib
case = sys.argv[1]
meta, arr = load(case)
disc = disc_from_golden(meta, arr)
try:
    A = pkg.assemble(form_of(meta), disc)
    print(case, "ok", _lib.last_kernel_times()[-1])
except Exception as e:
    print(case, "ERR", e)
