python tools/trace_call.py twisted 3 128 128 128 poisson full 2>&1 | grep "sg trace"
python - <<'PY'
import sys, time
sys.path.insert(0, ".")
import torch
import paper_1904_06971_b200 as pkg
from paper_1904_06971_b200 import _lib
from paper_1904_06971_b200.configs import CONFIGS
cfg = CONFIGS[5]
disc = pkg.make_discretization(cfg.geom(), cfg.p, cfg.spans)
fk = pkg.FormKind("mass")
s = torch.cuda.current_stream()
for it in range(3):
    res, _, _ = pkg.assemble_device(fk, disc, stream=s.cuda_stream); res.free()
torch.cuda.synchronize()
N = 6
ev = [torch.cuda.Event(enable_timing=True) for _ in range(N + 1)]
t0 = time.perf_counter()
ev[0].record(s)
walls = []
for i in range(N):
    a = time.perf_counter()
    res, _, _ = pkg.assemble_device(fk, disc, stream=s.cuda_stream)
    b = time.perf_counter()
    kt = _lib.last_kernel_times(); _lib.last_dmma_count(); res.sizes()
    c = time.perf_counter()
    res.free()
    d = time.perf_counter()
    ev[i + 1].record(s)
    walls.append((round(1e3 * (b - a), 3), round(1e3 * (c - b), 3), round(1e3 * (d - c), 3), round(_lib.last_timing()[0], 3), round(sum(t for _, t in kt), 3)))
torch.cuda.synchronize()
print("per job: (call wall, bookkeeping, free, device span, kernel sum)")
for i, w in enumerate(walls):
    print(w, "event-to-event", round(ev[i].elapsed_time(ev[i + 1]), 3))
PY
