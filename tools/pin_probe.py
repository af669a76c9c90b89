"""Host pinning cost probe: cudaHostAlloc / cudaHostRegister rates (development tool)."""
import ctypes
import glob
import time

import numpy as np
import torch

torch.cuda.init()
cands = glob.glob("/usr/local/cuda/lib64/libcudart.so*") + glob.glob("/usr/local/cuda/targets/*/lib/libcudart.so*")
rt = ctypes.CDLL(sorted(cands)[0])
libc = ctypes.CDLL("libc.so.6")
n = 2 << 30
for rep in range(2):
    p = ctypes.c_void_p()
    t = time.time(); rc = rt.cudaHostAlloc(ctypes.byref(p), ctypes.c_size_t(n), 0); dt = time.time() - t
    print(f"cudaHostAlloc 2 GiB: rc={rc} {n / dt / 1e9:.1f} GB/s ({dt*1e3:.0f} ms)")
    t = time.time(); rt.cudaFreeHost(p); print(f"  cudaFreeHost {1e3*(time.time()-t):.0f} ms")
for huge in (False, True):
    a = np.empty(n, dtype=np.uint8)
    if huge:
        addr = a.ctypes.data; al = (addr + (1 << 21) - 1) & ~((1 << 21) - 1)
        libc.madvise(ctypes.c_void_p(al), ctypes.c_size_t(n - (al - addr) - (1 << 21)), 14)
    t = time.time(); rc = rt.cudaHostRegister(ctypes.c_void_p(a.ctypes.data), ctypes.c_size_t(n), 0); dt = time.time() - t
    print(f"cudaHostRegister fresh 2 GiB huge={huge}: rc={rc} {n / dt / 1e9:.1f} GB/s ({dt*1e3:.0f} ms)")
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    t = time.time(); rt.cudaMemcpy(ctypes.c_void_p(a.ctypes.data), ctypes.c_void_p(d.data_ptr()), ctypes.c_size_t(n), 2); dt = time.time() - t
    print(f"  D2H into registered: {n / dt / 1e9:.1f} GB/s")
    t = time.time(); rt.cudaHostUnregister(ctypes.c_void_p(a.ctypes.data)); print(f"  unregister {1e3*(time.time()-t):.0f} ms")
# pre-faulted buffer (pages already mapped): registration cost alone
a = np.empty(n, dtype=np.uint8)
a[::4096] = 1
t = time.time(); rc = rt.cudaHostRegister(ctypes.c_void_p(a.ctypes.data), ctypes.c_size_t(n), 0); dt = time.time() - t
print(f"cudaHostRegister pre-faulted 2 GiB: rc={rc} {n / dt / 1e9:.1f} GB/s ({dt*1e3:.0f} ms)")
rt.cudaHostUnregister(ctypes.c_void_p(a.ctypes.data))
t = time.time(); rc = rt.cudaHostRegister(ctypes.c_void_p(a.ctypes.data), ctypes.c_size_t(n), 0); dt = time.time() - t
print(f"cudaHostRegister again (re-register) 2 GiB: rc={rc} {n / dt / 1e9:.1f} GB/s ({dt*1e3:.0f} ms)")
