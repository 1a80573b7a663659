"""Standalone check of the 3xTF32 tcgen05 matmul (run under `timeout`)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1801_04348_b200 import _lib, binding, programs
from oracle import oracle

kind = programs.original("matmul")
for n in [int(x) for x in (sys.argv[1:] or ["256", "512", "1024"])]:
    rng = np.random.default_rng(n)
    a = rng.uniform(-1, 1, (n, n)).astype(np.float32)
    b = rng.uniform(-1, 1, (n, n)).astype(np.float32)
    c = rng.uniform(-1, 1, (n, n)).astype(np.float32)
    P = {"n": n, "B0": 128, "ub1": 8, "s": 16}
    L = binding.make_launch(kind, P, (), _lib.DTYPE_F32, extra_flags=_lib.FLAG_TF32X3)
    ta, tb, tc = (torch.from_numpy(x.reshape(-1)).cuda() for x in (a, b, c))
    t0 = time.time()
    _lib.launch(L, [ta.data_ptr(), tb.data_ptr(), tc.data_ptr()])
    torch.cuda.synchronize()
    print("n", n, "launch+sync %.3fs" % (time.time() - t0), flush=True)
    got = tc.cpu().numpy().reshape(n, n).astype(np.float64)
    if n <= 2048:
        want = oracle.run("matmul", P, {"a": a, "b": b, "c": c})["c"]
        scale = (np.abs(a.astype(np.float64)) @ np.abs(b.astype(np.float64))).max()
        err = np.abs(got - want).max() / scale
        ffma_like = np.abs(got - want).max()
        print("   normalised err %.3g (tol %.3g), max abs %.3g" % (err, max(1e-5 * n / 1024, 2 * n * 2**-24), ffma_like), flush=True)
    # timing
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    reps = 5
    for _ in range(reps):
        _lib.launch(L, [ta.data_ptr(), tb.data_ptr(), tc.data_ptr()], st.cuda_stream)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print("   %.3f ms  %.1f TFLOP/s (useful 2n^3)" % (ms, 2 * n**3 / ms / 1e9), flush=True)
