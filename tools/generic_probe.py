"""The generic path (generic.py: our emitted kernel) against the hand-written
leaves on the same family programs (development probe): run_program wall
time end to end (numpy int32 in, results out), and the emitted kernel's device
time per launch (CUDA events around the generic path's launches).

python tools/generic_probe.py
"""
import os
import sys
import time
import warnings

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1801_04348_b200 import generic, programs, run_program  # noqa: E402

warnings.simplefilter("ignore", RuntimeWarning)
CASES = [("reverse", {"N": 1 << 24, "s": 4, "B": 256}), ("jacobi", {"T": 10, "N": (1 << 24) + 2, "s": 4, "B": 256}),
         ("transpose", {"N": 4096, "s": 4, "B0": 32, "B1": 8}), ("matvec", {"N": 4096, "s": 1, "B": 256})]
rng = np.random.default_rng(1)
for fam, P in CASES:
    kind = programs.original(fam)
    shapes = programs.array_shapes(kind, P)
    arrays = {k: rng.integers(-1000, 1000, size=s).astype(np.int32) for k, s in shapes.items()}
    text = programs.source(fam)
    res = {}
    for label, kw in (("leaf", {}), ("generic", {"via_generic": True})):
        run_program(text, P, arrays, **kw)
        torch.cuda.synchronize()
        t = time.perf_counter()
        out = run_program(text, P, arrays, **kw)
        torch.cuda.synchronize()
        res[label] = (time.perf_counter() - t, out)
    same = all(np.array_equal(np.asarray(res["leaf"][1][k]).reshape(-1), np.asarray(res["generic"][1][k]).reshape(-1))
               for k in res["leaf"][1])
    print("%-9s leaf %8.2f ms  generic %8.2f ms (%s, %d launches, mode %s, flat %s)" % (
        fam, res["leaf"][0] * 1e3, res["generic"][0] * 1e3, "same" if same else "DIFFER", generic.last.launches,
        generic.last.mode, generic.last.flat), flush=True)
