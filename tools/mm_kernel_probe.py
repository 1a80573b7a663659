"""FP32 matmul TMA leaves at several n and at the 8-rank share of n = 8192
(development probe): "big" = the 128 x 128 tile (B0 = 128, ub1*s = 128), "mid" =
the 128 x 64 tile (ub1*s = 64); a ":1" suffix selects the row-major-a kernels
(PK_MM_ROWA=1) instead of the a^T-slab ones.  Prints time, TFLOP/s and whether the bits of c
agree between the kernels (they must: same fma sequence).  PK_MM_KERNEL is set
to the name for kernels the library selects by that knob (tuning aid).

python tools/mm_kernel_probe.py [kernels=big,mid] [sizes=2048,4096,8192,8192/8]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1801_04348_b200 import _lib, binding, cases, programs  # noqa: E402

kernels = sys.argv[1].split(",") if len(sys.argv) > 1 else ["big", "mid"]
sizes = sys.argv[2].split(",") if len(sys.argv) > 2 else ["2048", "4096", "8192", "8192/8"]
kind = programs.original("matmul")
st = torch.cuda.current_stream()
for sz in sizes:
    n, share = (int(sz.split("/")[0]), int(sz.split("/")[1])) if "/" in sz else (int(sz), 1)
    g = torch.Generator(device="cuda").manual_seed(n)
    a, b, c0 = (torch.rand(n * n, device="cuda", generator=g) - 0.5 for _ in range(3))
    rows = n // share
    ref = None
    for k in kernels:
        P = {"n": n, "B0": 128, "ub1": 4 if k.startswith("mid") else 8, "s": 16}
        L = binding.make_launch(kind, P, cases.select(kind, P).applied, _lib.DTYPE_F32, lo=0,
                                hi=rows if share > 1 else 0)
        os.environ["PK_MM_KERNEL"] = k
        # "big:1" / "mid:1": a's rows as they lie (PK_MM_ROWA=1); default: the a^T-slab kernels
        # "big1p" / "big2": force the 128 x 128 tile at one / two CTAs per SM
        # (PK_MM_TILE); plain "big" lets the library choose by the tile count
        if k.startswith("big1p") or k.startswith("big2"):
            os.environ["PK_MM_TILE"] = "big1p" if k.startswith("big1p") else "big"
        else:
            os.environ.pop("PK_MM_TILE", None)
        if ":" in k:
            os.environ["PK_MM_ROWA"] = k.split(":")[1]
        else:
            os.environ.pop("PK_MM_ROWA", None)
        c = c0.clone()
        _lib.launch(L, [a.data_ptr(), b.data_ptr(), c.data_ptr()], st.cuda_stream)
        torch.cuda.synchronize()
        same = "ref" if ref is None else ("bits equal" if torch.equal(c[: rows * n], ref[: rows * n]) else "BITS DIFFER")
        if ref is None:
            ref = c.clone()
        reps = 30 if n * rows <= 2048 * 2048 else 8
        for _ in range(2):
            _lib.launch(L, [a.data_ptr(), b.data_ptr(), c.data_ptr()], st.cuda_stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(st)
        for _ in range(reps):
            _lib.launch(L, [a.data_ptr(), b.data_ptr(), c.data_ptr()], st.cuda_stream)
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        tf = 2 * rows * n * n / ms / 1e9
        print("n=%d rows=%d %-5s %.4f ms %.2f TFLOP/s (%.3f of 74.45)  %s" % (n, rows, k, ms, tf, tf / 74.45, same),
              flush=True)
    del a, b, c0, ref, c
    os.environ.pop("PK_MM_KERNEL", None)
