"""Fresh-memory copy rates: malloc'd numpy vs mmap + MADV_HUGEPAGE (development probe)."""
import mmap
import time

import numpy as np
import torch

n = 64 << 20  # float32 elements (256 MB)
src = np.random.default_rng(0).random(n, dtype=np.float32)
print("THP mode:", open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip())
for trial in range(3):
    t0 = time.perf_counter()
    dst = torch.empty(n, dtype=torch.float32)
    dst.copy_(torch.from_numpy(src))
    t1 = time.perf_counter()
    mm = mmap.mmap(-1, n * 4, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    mm.madvise(mmap.MADV_HUGEPAGE)
    arr = np.frombuffer(mm, dtype=np.float32)
    torch.from_numpy(arr).copy_(torch.from_numpy(src))
    t2 = time.perf_counter()
    print("torch.empty+copy %.1f ms | mmap THP + copy %.1f ms" % ((t1 - t0) * 1e3, (t2 - t1) * 1e3), flush=True)
    del arr, dst
    mm.close()
