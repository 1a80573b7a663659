"""Quick per-family device timing (development aid; bench.py is the contract).

python tools/quick_bench.py [family ...]
"""

import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1801_04348_b200 import _lib, binding, cases, programs  # noqa: E402
from paper_1801_04348_b200 import machine as machine_mod  # noqa: E402

CONFIGS = {
    "reverse": [({"N": 1 << 30, "s": 16, "B": 256}, 8 * (1 << 30)),
                ({"N": 1 << 30, "s": 4, "B": 1024}, 8 * (1 << 30)),
                ({"N": 1 << 30, "s": 64, "B": 128}, 8 * (1 << 30))],
    "transpose": [({"N": 32768, "s": 4, "B0": 32, "B1": 8}, 8 * 32768**2),
                  ({"N": 32768, "s": 8, "B0": 64, "B1": 8}, 8 * 32768**2),
                  ({"N": 32768, "s": 2, "B0": 16, "B1": 16}, 8 * 32768**2)],
    "jacobi": [({"T": 10, "N": (1 << 28) + 2, "s": s, "B": b}, 10 * 8 * (1 << 28))
               for (b, s) in [(256, 16), (1024, 4), (256, 8), (256, 32), (128, 32), (512, 8), (128, 16)]],
    "jacobi2d": [({"T": 10, "N": 16386, "s": s, "B0": b0, "B1": b1}, 10 * 8 * 16384**2)
                 for (b0, b1, s) in [(32, 8, 16), (64, 4, 32), (16, 16, 32), (8, 32, 16), (16, 32, 16),
                                     (8, 64, 16), (32, 8, 32), (16, 8, 64), (8, 16, 64)]],
    "matvec": [({"N": 32768, "s": 1, "B": 256}, 4 * 32768**2),
               ({"N": 32768, "s": 4, "B": 1024}, 4 * 32768**2)],
    "matmul": [({"n": 8192, "B0": 128, "ub1": 8, "s": 16}, 2 * 8192**3),
               ({"n": 8192, "B0": 64, "ub1": 8, "s": 16}, 2 * 8192**3),
               ({"n": 8192, "B0": 128, "ub1": 8, "s": 8}, 2 * 8192**3),
               ({"n": 2048, "B0": 128, "ub1": 8, "s": 16}, 2 * 2048**3),
               ({"n": 1024, "B0": 8, "ub1": 16, "s": 4}, 2 * 1024**3)],
    "addition": [({"N": 32768, "B0": 8, "B1": 128}, 12 * 32768**2)],
}


def main():
    fams = sys.argv[1:] or list(CONFIGS)
    mv = machine_mod.live()
    print("machine", mv.values, mv.props["name"], mv.props["sm_count"])
    dev = torch.device("cuda")
    for fam in fams:
        kind = programs.original(fam)
        for params, work in CONFIGS[fam]:
            sel = cases.select(kind, params, mv)
            dtype = _lib.DTYPE_F32 if fam == "matmul" else _lib.DTYPE_I32
            L = binding.make_launch(kind, params, sel.applied, dtype)
            shapes = programs.array_shapes(kind, params)
            bufs = []
            for a in programs.FAMILIES[fam].arrays:
                n = 1
                for d in shapes[a.name]:
                    n *= d
                if dtype == _lib.DTYPE_F32:
                    bufs.append(torch.rand(n, device=dev) - 0.5)
                else:
                    bufs.append(torch.randint(-1000, 1000, (n,), dtype=torch.int32, device=dev))
            ptrs = [b.data_ptr() for b in bufs]
            st = torch.cuda.current_stream().cuda_stream
            for _ in range(2):
                _lib.launch(L, ptrs, st)
            torch.cuda.synchronize()
            reps = 3
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                _lib.launch(L, ptrs, st)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            unit = "GFLOP/s" if fam == "matmul" else "GB/s"
            print("%-9s case %d %-28s %-40s %9.3f ms  %10.1f %s" % (
                fam, sel.index, ",".join(sel.applied) or "-", params, ms, work / ms / 1e6, unit), flush=True)
            del bufs
            torch.cuda.empty_cache()


if __name__ == "__main__":
    t = time.time()
    main()
    print("total %.1fs" % (time.time() - t))
