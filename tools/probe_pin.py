"""Probe: cost of pinned host buffers (torch caching allocator vs
mmap + cudaHostRegister) -- the first-call overhead of the file pipeline."""
import ctypes
import mmap
import time

import numpy as np
import torch

torch.cuda.init()
torch.empty(1, device="cuda")
for gb in (0.5, 1, 2, 4):
    n = int(gb * (1 << 30))
    t = time.perf_counter()
    a = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    t1 = time.perf_counter() - t
    t = time.perf_counter()
    a.fill_(1)
    t2 = time.perf_counter() - t
    del a
    cudart = ctypes.CDLL("libcudart.so.12") if False else None
    t = time.perf_counter()
    m = mmap.mmap(-1, n, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS | getattr(mmap, "MAP_POPULATE", 0))
    t3 = time.perf_counter() - t
    buf = np.frombuffer(m, dtype=np.uint8)
    t = time.perf_counter()
    rc = torch.cuda.cudart().cudaHostRegister(buf.ctypes.data, n, 0)
    t4 = time.perf_counter() - t
    torch.cuda.cudart().cudaHostUnregister(buf.ctypes.data)
    del buf
    m.close()
    print(f"{gb} GiB: torch pinned alloc {t1:.3f}s, first touch {t2:.3f}s; mmap populate {t3:.3f}s, "
          f"cudaHostRegister {t4:.3f}s rc={rc}", flush=True)
