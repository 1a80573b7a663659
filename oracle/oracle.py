"""TEST INFRASTRUCTURE ONLY -- numpy/ctypes front end of the CPU oracle.

Wraps oracle/libpk_oracle.so (pk_oracle.c), the C restatement of the
reference interpreter's semantics (parakern.interp.run_program,
/root/reference/pkg/src/parakern/interp.py:215-225) for the seven program
families.  Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline
and --impl reference) may import this module; the product package never
does.

Pinning: tests/test_oracle.py checks every function here against the golden
vectors of tests/golden/ (generated from the reference interpreter itself by
tests/golden/make_golden.py) and the hand-computed vectors of the
reference's own tests (pkg/tests/test_interp.py:43-88).

run(family, params, arrays) mirrors run_program: params in the ORIGINAL
program's names (a granularity program is passed with s=1, and the merged
addition with merged=True), arrays as numpy arrays in declaration shape;
returns a dict of fresh arrays.  Integer families return int32; matmul /
matvec with float inputs return float64 (the reference's Python floats).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libpk_oracle.so")

_lib = None


def build() -> str:
    src = os.path.join(HERE, "pk_oracle.c")
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB)
        i64 = ctypes.c_int64
        P = ctypes.c_void_p
        sig = {
            "pko_reverse_i32": [i64, i64, i64, P, P],
            "pko_transpose_u32": [i64, i64, i64, i64, P, P],
            "pko_jacobi1d_i32": [i64, i64, i64, i64, P],
            "pko_jacobi2d_i32": [i64, i64, i64, i64, i64, P],
            "pko_matvec_i32": [i64, i64, i64, P, P, P],
            "pko_matvec_f64": [i64, i64, i64, P, P, P],
            "pko_matmul_i32": [i64, i64, i64, i64, P, P, P],
            "pko_matmul_f64": [i64, i64, i64, i64, P, P, P],
            "pko_matmul_f64_rows": [i64, i64, i64, i64, i64, i64, P, P, P],
            "pko_addition_i32": [i64, i64, i64, P, P, P],
        }
        for name, args in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = ctypes.c_int
        L.pko_num_threads.restype = ctypes.c_int
        L.pko_set_threads.argtypes = [ctypes.c_int]
        _lib = L
    return _lib


def threads() -> int:
    return int(lib().pko_num_threads())


def set_threads(n: int) -> None:
    lib().pko_set_threads(int(n))


def _p(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def _check(rc: int, what: str) -> None:
    if rc == 3:
        raise ZeroDivisionError(what)
    if rc != 0:
        raise RuntimeError("%s: oracle error %d" % (what, rc))


def _i32(x, shape):
    a = np.ascontiguousarray(np.asarray(x), dtype=np.int32)
    return a.reshape(shape).copy()


def _is_float(x) -> bool:
    return x is not None and np.issubdtype(np.asarray(x).dtype, np.floating)


def matmul_rows_f64(params: dict, r0: int, r1: int, a: np.ndarray, b: np.ndarray, c: np.ndarray) -> None:
    """Rows [r0, r1) of the matmul program in binary64 (in place on c, float64
    n x n; a, b float32 n x n) -- a bounded sample of one full run."""
    P = {k: int(v) for k, v in params.items()}
    assert a.dtype == np.float32 and b.dtype == np.float32 and c.dtype == np.float64
    _check(lib().pko_matmul_f64_rows(P["n"], P["B0"], P["ub1"], P["s"], r0, r1, _p(a), _p(b), _p(c)), "matmul")


def run(family: str, params: dict, arrays: dict | None = None, *, merged: bool = False) -> dict:
    arrays = arrays or {}
    L = lib()
    P = {k: int(v) for k, v in params.items()}
    if family == "reverse":
        N = P["N"]
        a = _i32(arrays.get("a", np.zeros(N)), (N,)) if not _is_float(arrays.get("a")) else None
        if a is None:  # float words move as bit patterns
            a = np.ascontiguousarray(arrays["a"], dtype=np.float32).view(np.int32).copy()
        c = _i32(arrays.get("c", np.zeros(N)), (N,)) if not _is_float(arrays.get("c")) else \
            np.ascontiguousarray(arrays["c"], dtype=np.float32).view(np.int32).copy()
        _check(L.pko_reverse_i32(N, P["s"], P["B"], _p(a), _p(c)), "reverse")
        if _is_float(arrays.get("a")):
            return {"a": a.view(np.float32), "c": c.view(np.float32)}
        return {"a": a, "c": c}
    if family == "transpose":
        N = P["N"]
        fl = _is_float(arrays.get("a"))
        a = np.ascontiguousarray(arrays.get("a", np.zeros((N, N))), dtype=np.float32 if fl else np.int32)
        a = a.reshape(N, N).view(np.uint32).copy()
        c0 = arrays.get("c", np.zeros(N * N))
        c = np.ascontiguousarray(c0, dtype=np.float32 if fl else np.int32).reshape(N * N).view(np.uint32).copy()
        _check(L.pko_transpose_u32(N, P["s"], P["B0"], P["B1"], _p(a), _p(c)), "transpose")
        vt = np.float32 if fl else np.int32
        return {"a": a.view(vt), "c": c.view(vt)}
    if family == "jacobi":
        N = P["N"]
        a = _i32(arrays.get("a", np.zeros(2 * N)), (2 * N,))
        _check(L.pko_jacobi1d_i32(P["T"], N, P["s"], P["B"], _p(a)), "jacobi")
        return {"a": a}
    if family == "jacobi2d":
        N = P["N"]
        a = _i32(arrays.get("a", np.zeros((2 * N, N))), (2 * N, N))
        _check(L.pko_jacobi2d_i32(P["T"], N, P["s"], P["B0"], P["B1"], _p(a)), "jacobi2d")
        return {"a": a}
    if family == "matvec":
        N = P["N"]
        if any(_is_float(arrays.get(k)) for k in ("a", "x", "y")):
            a = np.ascontiguousarray(arrays.get("a", np.zeros((N, N))), dtype=np.float32).reshape(N, N)
            x = np.ascontiguousarray(arrays.get("x", np.zeros(N)), dtype=np.float32).reshape(N)
            y = np.ascontiguousarray(arrays.get("y", np.zeros(N)), dtype=np.float64).reshape(N).copy()
            _check(L.pko_matvec_f64(N, P["s"], P["B"], _p(a), _p(x), _p(y)), "matvec")
            return {"a": a.copy(), "x": x.copy(), "y": y}
        a = _i32(arrays.get("a", np.zeros((N, N))), (N, N))
        x = _i32(arrays.get("x", np.zeros(N)), (N,))
        y = _i32(arrays.get("y", np.zeros(N)), (N,))
        _check(L.pko_matvec_i32(N, P["s"], P["B"], _p(a), _p(x), _p(y)), "matvec")
        return {"a": a, "x": x, "y": y}
    if family == "matmul":
        n = P["n"]
        if any(_is_float(arrays.get(k)) for k in ("a", "b", "c")):
            a = np.ascontiguousarray(arrays.get("a", np.zeros((n, n))), dtype=np.float32).reshape(n, n)
            b = np.ascontiguousarray(arrays.get("b", np.zeros((n, n))), dtype=np.float32).reshape(n, n)
            c = np.ascontiguousarray(arrays.get("c", np.zeros((n, n))), dtype=np.float64).reshape(n, n).copy()
            _check(L.pko_matmul_f64(n, P["B0"], P["ub1"], P["s"], _p(a), _p(b), _p(c)), "matmul")
            return {"a": a.copy(), "b": b.copy(), "c": c}
        a = _i32(arrays.get("a", np.zeros((n, n))), (n, n))
        b = _i32(arrays.get("b", np.zeros((n, n))), (n, n))
        c = _i32(arrays.get("c", np.zeros((n, n))), (n, n))
        _check(L.pko_matmul_i32(n, P["B0"], P["ub1"], P["s"], _p(a), _p(b), _p(c)), "matmul")
        return {"a": a, "b": b, "c": c}
    if family == "addition":
        N = P["N"]
        a = _i32(arrays.get("a", np.zeros(N * N)), (N * N,))
        b = _i32(arrays.get("b", np.zeros(N * N)), (N * N,))
        c = _i32(arrays.get("c", np.zeros(N * N)), (N * N,))
        if merged:
            # granularity-merged program (strategies.py:213-262): one store,
            # j < (N/B1)*B1 -- restated directly (small sizes only)
            B0, B1 = P["B0"], P["B1"]
            if B0 == 0 or B1 == 0:
                raise ZeroDivisionError("addition")
            I = max(0, N // B0) * B0 if B0 > 0 else 0
            J = max(0, N // B1) * B1 if B1 > 0 else 0
            for i in range(min(I, N)):
                for j in range(min(J, N)):
                    c[i * N + j] = np.int32(int(a[i * N + j]) + int(b[i * N + j]))
            return {"a": a, "b": b, "c": c}
        _check(L.pko_addition_i32(N, P["B0"], P["B1"], _p(a), _p(b), _p(c)), "addition")
        return {"a": a, "b": b, "c": c}
    raise KeyError(family)
