"""FP32 matmul leaf times per tile (B0, ub1, s) at several n (development probe)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1801_04348_b200 import _lib, binding, cases, programs  # noqa: E402

kind = programs.original("matmul")
for n in (1024, 2048, 4096, 8192):
    bufs = [torch.rand(n * n, device="cuda") - 0.5 for _ in range(3)]
    ptrs = [b.data_ptr() for b in bufs]
    st = torch.cuda.current_stream()
    for B0, ub1, s in ((128, 8, 16), (64, 8, 8)):
        P = {"n": n, "B0": B0, "ub1": ub1, "s": s}
        L = binding.make_launch(kind, P, cases.select(kind, P).applied, _lib.DTYPE_F32)
        for _ in range(2):
            _lib.launch(L, ptrs, st.cuda_stream)
        reps = 20 if n <= 2048 else 5
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(st)
        for _ in range(reps):
            _lib.launch(L, ptrs, st.cuda_stream)
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        print("n=%d tile %dx%d: %.3f ms %.1f TFLOP/s" % (n, B0, ub1 * s, ms, 2 * n**3 / ms / 1e9), flush=True)
    del bufs
