"""Matmul schedules at n = 8192 and an 8-rank share: the order-preserving
split (default) vs lockstep pieces (PK_MM_SCHED=pieces, PK_MM_PIECES=D,
PK_MM_PGROUP=G); CUDA-event times and an exactness check (development probe;
run under ncu --metrics dram__bytes_read.sum for the traffic).  The pieces
schedule was measured slower and removed from the
library; the environment variables are then ignored."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1801_04348_b200 import _lib, binding, cases, programs  # noqa: E402

configs = [c.split(":") for c in (sys.argv[1] if len(sys.argv) > 1 else "split::,pieces:4:592,pieces:8:592").split(",")]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
kind = programs.original("matmul")
for n, rows in ((8192, 8192), (8192, 1024)):
    P = {"n": n, "B0": 128, "ub1": 8, "s": 16}
    L = binding.make_launch(kind, P, cases.select(kind, P).applied, _lib.DTYPE_F32, lo=0, hi=rows)
    g = torch.Generator(device="cuda").manual_seed(1)
    a, b = (torch.rand(n * n, device="cuda", generator=g) - 0.5 for _ in range(2))  # bit-identity needs order
    c = torch.zeros(n * n, device="cuda")
    ptrs = [a.data_ptr(), b.data_ptr(), c.data_ptr()]
    ref = None
    st = torch.cuda.current_stream()
    for sched, D, G in configs:
        for k in ("PK_MM_SCHED", "PK_MM_PIECES", "PK_MM_PGROUP"):
            os.environ.pop(k, None)
        if sched != "split":
            os.environ["PK_MM_SCHED"] = sched
            if D:
                os.environ["PK_MM_PIECES"] = D
            if G:
                os.environ["PK_MM_PGROUP"] = G
        c.zero_()
        _lib.launch(L, ptrs, st.cuda_stream)
        torch.cuda.synchronize()
        if ref is None:
            ref = c.clone()
        exact = bool(torch.equal(c, ref))
        _lib.launch(L, ptrs, st.cuda_stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(st)
        for _ in range(reps):
            _lib.launch(L, ptrs, st.cuda_stream)
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        print("rows=%d %-7s D=%-2s G=%-4s %.3f ms %.1f TFLOP/s exact=%s" % (rows, sched, D, G, ms,
              2 * rows * n * n / ms / 1e9, exact), flush=True)
