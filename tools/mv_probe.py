import sys, os
sys.path.insert(0, "/root/repo")
import torch, numpy as np
from paper_1801_04348_b200 import _lib, binding, cases, programs
kind = programs.original("matvec")
for N, vals in ((64, "ones"), (1024, "ones"), (1024, "rand"), (32768, "rand")):
    P = {"N": N, "s": 1, "B": 512 if N >= 512 else N}
    L = binding.make_launch(kind, P, cases.select(kind, P).applied, _lib.DTYPE_F32)
    if vals == "ones":
        a = torch.ones(N * N, device="cuda"); x = torch.ones(N, device="cuda")
    else:
        g = torch.Generator(device="cuda").manual_seed(1)
        a = torch.rand(N * N, device="cuda", generator=g) - 0.5; x = torch.rand(N, device="cuda", generator=g) - 0.5
    y = torch.zeros(N, device="cuda")
    _lib.launch(L, [a.data_ptr(), x.data_ptr(), y.data_ptr()], torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    want = a.view(N, N).double() @ x.double()
    err = ((y.double() - want).abs() / want.abs().clamp_min(1e-30))
    print(N, vals, "y[:4]", y[:4].tolist(), "want", want[:4].tolist(), "max rel err", err.max().item(), flush=True)
# timing at the BASELINE-proposed size
N = 32768
P = {"N": N, "s": 1, "B": 512}
L = binding.make_launch(kind, P, cases.select(kind, P).applied, _lib.DTYPE_F32)
a = torch.rand(N * N, device="cuda") - 0.5; x = torch.rand(N, device="cuda"); y = torch.zeros(N, device="cuda")
ptrs = [a.data_ptr(), x.data_ptr(), y.data_ptr()]
st = torch.cuda.current_stream()
for _ in range(3):
    _lib.launch(L, ptrs, st.cuda_stream)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); e0.record(st)
for _ in range(20):
    _lib.launch(L, ptrs, st.cuda_stream)
e1.record(st); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print("float32 matvec N=32768: %.3f ms  %.1f GB/s" % (ms, (4 * N * N + 8 * N) / ms / 1e6))
