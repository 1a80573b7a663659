"""Sweep the matmul raster group (PK_MM_GROUP) at n = 8192, an 8-rank share
(1024 rows) and n = 2048: CUDA-event times per launch (development probe;
run under ncu with --metrics dram__bytes_read.sum,dram__bytes_write.sum for
the traffic side).  python tools/mm_group_probe.py [groups] [reps] [s] [n/rows,...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1801_04348_b200 import _lib, binding, cases, programs  # noqa: E402

groups = [int(g) for g in (sys.argv[1].split(",") if len(sys.argv) > 1 else "4,8,12,16,24,32".split(","))]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
s_tile = int(sys.argv[3]) if len(sys.argv) > 3 else 16  # 16: the 128 x 128 tile, 8: 128 x 64
shapes = ((8192, 8192), (8192, 1024), (2048, 2048)) if len(sys.argv) <= 4 else \
    tuple(tuple(int(v) for v in x.split("/")) for x in sys.argv[4].split(","))
kind = programs.original("matmul")
for n, rows in shapes:
    P = {"n": n, "B0": 128, "ub1": 8, "s": s_tile}
    L = binding.make_launch(kind, P, cases.select(kind, P).applied, _lib.DTYPE_F32, lo=0, hi=rows)
    bufs = [torch.rand(n * n, device="cuda") - 0.5 for _ in range(3)]
    ptrs = [b.data_ptr() for b in bufs]
    st = torch.cuda.current_stream()
    for g in groups:
        os.environ["PK_MM_GROUP"] = str(g)
        for _ in range(2):
            _lib.launch(L, ptrs, st.cuda_stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(st)
        for _ in range(reps):
            _lib.launch(L, ptrs, st.cuda_stream)
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        print("n=%d rows=%d group=%2d  %.3f ms  %.1f TFLOP/s" % (n, rows, g, ms, 2 * rows * n * n / ms / 1e9),
              flush=True)
    del bufs
