"""Small run_program host-path calls with a watchdog (development aid)."""
import faulthandler
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
faulthandler.dump_traceback_later(int(os.environ.get("WATCHDOG", "60")), exit=True)
import numpy as np  # noqa: E402

from paper_1801_04348_b200 import programs, run_program  # noqa: E402

for n in (64, 512, 2048, 8192):
    P = {"n": n, "B0": 128 if n >= 128 else 16, "ub1": 8, "s": 16 if n >= 128 else 1}
    a = np.ones((n, n), np.float32)
    t0 = time.perf_counter()
    out = run_program(programs.source("matmul"), P, {"a": a, "b": a, "c": np.zeros((n, n), np.float32)})
    print("n", n, "ok", float(out["c"][0, 0]), "%.1f ms" % ((time.perf_counter() - t0) * 1e3), flush=True)
for N in (1 << 10, 1 << 24):
    a = np.arange(N, dtype=np.int32)
    t0 = time.perf_counter()
    out = run_program(programs.source("reverse"), {"N": N, "s": 4, "B": 256}, {"a": a})
    print("reverse", N, bool((out["c"] == a[::-1]).all()), "%.1f ms" % ((time.perf_counter() - t0) * 1e3), flush=True)
