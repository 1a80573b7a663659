"""pk_run_host_io variants at n = 8192: which host copies cost what (development probe)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1801_04348_b200 import _lib, binding, cases, programs, run_program  # noqa: E402

n = 8192
P = {"n": n, "B0": 128, "ub1": 8, "s": 16}
rng = np.random.default_rng(0)
a, b = (rng.random((n, n), dtype=np.float32) for _ in range(2))
c = np.zeros((n, n), np.float32)
kind = programs.original("matmul")
L = binding.make_launch(kind, P, cases.select(kind, P).applied, _lib.DTYPE_F32)
fresh = lambda: torch.empty(n * n, dtype=torch.float32).numpy()  # noqa: E731
warm = [fresh() for _ in range(3)]
for w in warm:
    w[:] = 0


def t(label, outs_fn, reps=4):
    for i in range(reps):
        outs = outs_fn()
        t0 = time.perf_counter()
        _lib.run_host_io(L, [a.ctypes.data, b.ctypes.data, c.ctypes.data], [o.ctypes.data if o is not None else 0
                                                                            for o in outs], [n * n] * 3, 0)
        dt = time.perf_counter() - t0
        if i:
            print("%-40s %.2f ms" % (label, dt * 1e3), flush=True)


t("c fresh only", lambda: [None, None, fresh()])
t("c warm only", lambda: [None, None, warm[2]])
t("a, b, c fresh", lambda: [fresh(), fresh(), fresh()])
t("a, b, c warm", lambda: warm)
text = programs.source("matmul")
for i in range(4):
    t0 = time.perf_counter()
    run_program(text, P, {"a": a, "b": b, "c": c})
    print("run_program %.2f ms" % ((time.perf_counter() - t0) * 1e3), flush=True)
import cProfile, pstats  # noqa: E401,E402
pr = cProfile.Profile()
pr.enable()
run_program(text, P, {"a": a, "b": b, "c": c})
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(12)
