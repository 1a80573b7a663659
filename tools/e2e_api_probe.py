"""Time run_program with numpy host arrays at n = 8192 (the drop-in API's
host path) beside pk_run_host on pinned buffers (development probe)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch

from paper_1801_04348_b200 import _lib, binding, cases, programs, run_program

n = 8192
P = {"n": n, "B0": 128, "ub1": 8, "s": int(sys.argv[1]) if len(sys.argv) > 1 else 16}
rng = np.random.default_rng(0)
a, b = (rng.random((n, n), dtype=np.float32) for _ in range(2))
c = np.zeros((n, n), np.float32)
text = programs.source("matmul")
for i in range(6):
    t0 = time.perf_counter()
    out = run_program(text, P, {"a": a, "b": b, "c": c})
    dt = time.perf_counter() - t0
    print("run_program numpy  %.2f ms  %.1f TFLOP/s" % (dt * 1e3, 2 * n**3 / dt / 1e12), flush=True)
kind = programs.original("matmul")
L = binding.make_launch(kind, P, cases.select(kind, P).applied, _lib.DTYPE_F32)
h = [torch.from_numpy(x.reshape(-1)).pin_memory() for x in (a, b, c)]
for i in range(4):
    t0 = time.perf_counter()
    _lib.run_host(L, [x.data_ptr() for x in h], 0)
    dt = time.perf_counter() - t0
    print("pk_run_host pinned %.2f ms  %.1f TFLOP/s" % (dt * 1e3, 2 * n**3 / dt / 1e12), flush=True)
# the native host path alone: pageable numpy in, fresh numpy out (pk_run_host_io)
out = np.empty((n, n), np.float32)
for i in range(4):
    t0 = time.perf_counter()
    _lib.run_host_io(L, [a.ctypes.data, b.ctypes.data, c.ctypes.data], [0, 0, out.ctypes.data], [n * n] * 3, 0)
    dt = time.perf_counter() - t0
    print("pk_run_host_io pageable %.2f ms  %.1f TFLOP/s" % (dt * 1e3, 2 * n**3 / dt / 1e12), flush=True)
import torch as _t  # noqa: E402
for i in range(3):
    t0 = time.perf_counter()
    x = _t.from_numpy(a).clone()
    y = _t.from_numpy(b).clone()
    dt = time.perf_counter() - t0
    print("clone a, b (512 MB) %.2f ms" % (dt * 1e3), flush=True)
