"""Time the binary64 (PK_DTYPE_F64) and int64 paths on device buffers (development probe)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1801_04348_b200 import _lib, binding, cases, machine, programs  # noqa: E402


def t(fam, P, dtype, tdt, reps=3):
    kind = programs.original(fam)
    mv = machine.live(0, elem_bytes=8)
    L = binding.make_launch(kind, P, cases.select(kind, P, mv).applied, dtype)
    shapes = programs.array_shapes(kind, P)
    bufs = []
    for a in programs.FAMILIES[fam].arrays:
        n = 1
        for d in shapes[a.name]:
            n *= d
        bufs.append((torch.rand(n, device="cuda", dtype=torch.float64) - 0.5).to(tdt))
    st = torch.cuda.current_stream()
    _lib.launch(L, [b.data_ptr() for b in bufs], st.cuda_stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record(st)
    for _ in range(reps):
        _lib.launch(L, [b.data_ptr() for b in bufs], st.cuda_stream)
    e1.record(st); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for n in (2048, 4096):
    P = {"n": n, "B0": 128, "ub1": 8, "s": 16}
    ms = t("matmul", P, _lib.DTYPE_F64, torch.float64)
    print("f64 matmul n=%d: %.2f ms  %.2f TFLOP/s" % (n, ms, 2 * n**3 / ms / 1e9), flush=True)
    P = {"n": n, "B0": 32, "ub1": 8, "s": 4}
    ms = t("matmul", P, _lib.DTYPE_F64, torch.float64)
    print("f64 matmul n=%d B0=32: %.2f ms  %.2f TFLOP/s" % (n, ms, 2 * n**3 / ms / 1e9), flush=True)
N = 32768
ms = t("matvec", {"N": N, "s": 1, "B": 512}, _lib.DTYPE_F64, torch.float64)
print("f64 matvec N=%d: %.3f ms  %.0f GB/s" % (N, ms, 8 * N * N / ms / 1e6))
ms = t("reverse", {"N": 1 << 29, "s": 16, "B": 256}, _lib.DTYPE_F64, torch.float64)
print("f64 reverse N=2^29: %.3f ms  %.0f GB/s" % (ms, 16 * (1 << 29) / ms / 1e6))
ms = t("transpose", {"N": 16384, "s": 8, "B0": 64, "B1": 8}, _lib.DTYPE_F64, torch.float64)
print("f64 transpose N=16384: %.3f ms  %.0f GB/s" % (ms, 16 * 16384**2 / ms / 1e6))
ms = t("addition", {"N": 16384, "B0": 8, "B1": 128}, _lib.DTYPE_F64, torch.float64)
print("f64 addition N=16384: %.3f ms  %.0f GB/s" % (ms, 24 * 16384**2 / ms / 1e6))
