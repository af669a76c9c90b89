"""Host-side copy-path probe: D2H to pinned, pinned -> fresh pageable, THP effect (development tool)."""
import ctypes
import mmap
import os
import threading
import time

import numpy as np
import torch

print("THP:", open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip(),
      "| defrag:", open("/sys/kernel/mm/transparent_hugepage/defrag").read().strip(), "| cpus:", os.cpu_count())
n = 2 << 30  # 2 GiB
dev = torch.empty(n, dtype=torch.uint8, device="cuda")
pin = torch.empty(n, dtype=torch.uint8, pin_memory=True)
torch.cuda.synchronize()
for _ in range(2):
    t = time.time(); pin.copy_(dev); torch.cuda.synchronize(); dt = time.time() - t
print(f"D2H device->pinned 2 GiB: {n / dt / 1e9:.1f} GB/s")
for _ in range(2):
    t = time.time(); dev.copy_(pin); torch.cuda.synchronize(); dt = time.time() - t
print(f"H2D pinned->device 2 GiB: {n / dt / 1e9:.1f} GB/s")
libc = ctypes.CDLL("libc.so.6")
src = pin.numpy()

def par_copy(dst, src, nt):
    per = (dst.size + nt - 1) // nt
    ths = [threading.Thread(target=lambda a, b: np.copyto(dst[a:b], src[a:b]), args=(k * per, min(dst.size, (k + 1) * per))) for k in range(nt)]
    [t.start() for t in ths]; [t.join() for t in ths]

for huge in (False, True):
    for nt in (1, 8, 16, 32):
        dst = np.empty(n, dtype=np.uint8)
        if huge:
            addr = dst.ctypes.data
            al = (addr + (1 << 21) - 1) & ~((1 << 21) - 1)
            libc.madvise(ctypes.c_void_p(al), ctypes.c_size_t(n - (al - addr) - (1 << 21)), 14)  # MADV_HUGEPAGE
        t = time.time(); par_copy(dst, src, nt); dt = time.time() - t
        t = time.time(); par_copy(dst, src, nt); dt2 = time.time() - t
        print(f"pinned->fresh pageable huge={huge} threads={nt}: first touch {n / dt / 1e9:.1f} GB/s, warm {n / dt2 / 1e9:.1f} GB/s")
        del dst
