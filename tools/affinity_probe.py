"""CPU affinity and copy-pool packing rate inside the Python process (is the host pool parallel?)."""
import os
import sys
import time

sys.path.insert(0, ".")
print("affinity before torch", sorted(os.sched_getaffinity(0)))
import torch  # noqa: E402

print("affinity after torch", sorted(os.sched_getaffinity(0)), "threads", torch.get_num_threads())
import paper_1904_06971_b200 as pkg  # noqa: E402

print("affinity after pkg", sorted(os.sched_getaffinity(0)))
import numpy as np  # noqa: E402

a = np.ones(2_165_248 // 8)
for _ in range(3):
    t = time.perf_counter()
    b = a.copy()
    print("numpy 2MB copy us", round((time.perf_counter() - t) * 1e6, 1))
