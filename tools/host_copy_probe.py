"""Host-side copy rates on the GPU box (development probe for the run_program
host path): numpy copy, torch (multi-threaded) copy into pinned memory,
pageable vs pinned H2D/D2H, and cudaHostRegister of a caller's buffer."""

import ctypes
import time

import numpy as np
import torch

MB = 1 << 20
n = 256 * MB // 4
src = np.random.default_rng(0).random(n, dtype=np.float32)
pinned = torch.empty(n, dtype=torch.float32, pin_memory=True)
dev = torch.empty(n, dtype=torch.float32, device="cuda")


def rate(label, fn, nbytes=n * 4, reps=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    print("%-44s %8.2f ms  %7.1f GB/s" % (label, dt * 1e3, nbytes / dt / 1e9), flush=True)


rate("numpy copy (fresh array)", lambda: src.copy())
dst = np.empty_like(src)
rate("np.copyto (existing array)", lambda: np.copyto(dst, src))
rate("torch copy_ into pinned (threads=%d)" % torch.get_num_threads(), lambda: pinned.copy_(torch.from_numpy(src)))
rate("torch clone to fresh", lambda: torch.from_numpy(src).clone())
rate("H2D from pinned", lambda: dev.copy_(pinned, non_blocking=True))
rate("H2D from pageable numpy", lambda: dev.copy_(torch.from_numpy(src)))
rate("D2H to pinned", lambda: pinned.copy_(dev, non_blocking=True))
rate("D2H to pageable", lambda: torch.from_numpy(dst).copy_(dev))

cudart = ctypes.CDLL("libcudart.so.12") if False else None
try:
    lib = ctypes.CDLL(torch.cuda.__file__.replace("cuda/__init__.py", "lib/libtorch_cuda.so"))
except OSError:
    lib = None
try:
    rt = ctypes.CDLL("libcudart.so")
except OSError:
    import glob
    cands = glob.glob("/usr/local/cuda/lib64/libcudart.so*")
    rt = ctypes.CDLL(cands[0]) if cands else None
if rt is not None:
    rt.cudaHostRegister.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint]
    rt.cudaHostUnregister.argtypes = [ctypes.c_void_p]
    buf = np.empty(n, np.float32)
    buf[:] = 1
    for _ in range(3):
        t0 = time.perf_counter()
        rc = rt.cudaHostRegister(buf.ctypes.data, n * 4, 0)
        t1 = time.perf_counter()
        rc2 = rt.cudaHostUnregister(buf.ctypes.data)
        t2 = time.perf_counter()
        print("cudaHostRegister 256 MiB rc=%d %.2f ms (%.1f GB/s), unregister rc=%d %.2f ms"
              % (rc, (t1 - t0) * 1e3, n * 4 / (t1 - t0) / 1e9, rc2, (t2 - t1) * 1e3), flush=True)
import os
print("cpus", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)), "torch threads", torch.get_num_threads())
