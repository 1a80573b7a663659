"""Randomised binary64 parity: every family on random parameters and random
binary64 data spanning 40 orders of magnitude (plus signed zeros, infinities
and subnormals), against numpy restatements of the programs in the
interpreter's own order -- c + a*b with two roundings, k ascending; Jacobi
sums left to right and c_div on Python floats (numpy's floor_divide is
CPython's fmod-based float floor division) -- bit for bit (NaNs as NaNs).
The fixed reference vectors are in tests/test_gpu_values.py; this widens
the draws (PK_FUZZ_DRAWS / PK_FUZZ_SEED as in test_gpu_fuzz.py)."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

DRAWS = int(os.environ.get("PK_FUZZ_DRAWS", 24))
SEED = int(os.environ.get("PK_FUZZ_SEED", 0))


def _values(rng, shape):
    v = rng.standard_normal(shape) * 10.0 ** rng.integers(-20, 20, size=shape)
    special = rng.random(shape) < 0.03
    v[special] = rng.choice([0.0, -0.0, np.inf, -np.inf, 5e-324, -1e308], size=int(special.sum()))
    return v


def _cdiv(s, d):
    q = np.floor_divide(np.abs(s), float(d))
    return np.where(s >= 0, q, -q)


def _params(family, rng):
    r = lambda lo, hi: int(rng.integers(lo, hi))  # noqa: E731
    if family == "reverse":
        return {"N": r(1, 3000), "s": r(1, 5), "B": r(1, 65)}
    if family == "transpose":
        return {"N": r(1, 90), "s": r(1, 4), "B0": r(1, 17), "B1": r(1, 17)}
    if family == "addition":
        B1 = r(1, 9)
        return {"N": 2 * B1 * r(1, 8), "B0": r(1, 9), "B1": B1}
    if family == "matvec":
        return {"N": r(1, 160), "s": r(1, 4), "B": r(1, 33)}
    if family == "matmul":
        return {"n": r(1, 100), "B0": r(1, 33), "ub1": r(1, 9), "s": r(1, 4)}
    if family == "jacobi":
        return {"T": r(0, 6), "N": r(2, 2000), "s": r(1, 5), "B": r(1, 65)}
    return {"T": r(0, 5), "N": r(2, 60), "s": r(1, 4), "B0": r(1, 9), "B1": r(1, 9)}


def _restate(family, P, arr):
    out = {k: v.copy() for k, v in arr.items()}
    if family == "reverse":
        N, t = P["N"], P["s"] * P["B"]
        Pc = (N // t) * t
        out["c"][N - Pc:] = arr["a"][:Pc][::-1]
    elif family == "transpose":
        N = P["N"]
        I, J = (N // P["B0"]) * P["B0"], (N // (P["s"] * P["B1"])) * P["s"] * P["B1"]
        out["c"].reshape(N, N)[:I, :J] = arr["a"].T[:I, :J]
    elif family == "addition":
        N = P["N"]
        I, J, h = (N // P["B0"]) * P["B0"], min((N // (2 * P["B1"])) * P["B1"], N // 2), N // 2
        a, b, c = (x.reshape(N, N) for x in (arr["a"], arr["b"], out["c"]))
        c[:I, :J] = a[:I, :J] + b[:I, :J]
        c[:I, h:h + J] = a[:I, h:h + J] + b[:I, h:h + J]
    elif family == "matvec":
        N, t = P["N"], P["s"] * P["B"]
        R = (N // t) * t
        for q in range(N):
            out["y"][:R] = out["y"][:R] + arr["a"][:R, q] * arr["x"][q]
    elif family == "matmul":
        n = P["n"]
        M = K = (n // P["B0"]) * P["B0"]
        Nc = (n // (P["ub1"] * P["s"])) * P["ub1"] * P["s"]
        for kk in range(K):
            out["c"][:M, :Nc] = out["c"][:M, :Nc] + np.outer(arr["a"][:M, kk], arr["b"][kk, :Nc])
    elif family == "jacobi":
        N, t = P["N"], P["s"] * P["B"]
        Pc = max(0, (N - 2) // t) * t
        a = out["a"]
        for step in range(P["T"]):
            src, dst = (a[N:], a[:N]) if step % 2 == 0 else (a[:N], a[N:])
            if Pc:
                dst[1:Pc + 1] = _cdiv((src[0:Pc] + src[1:Pc + 1]) + src[2:Pc + 2], 3)
    else:
        N = P["N"]
        I = max(0, (N - 2) // P["B0"]) * P["B0"]
        J = max(0, (N - 2) // (P["s"] * P["B1"])) * P["s"] * P["B1"]
        a = out["a"]
        for step in range(P["T"]):
            src, dst = (a[:N], a[N:]) if step % 2 == 0 else (a[N:], a[:N])
            if I and J:
                s = src[0:I, 1:J + 1] + src[2:I + 2, 1:J + 1]
                s = s + src[1:I + 1, 0:J]
                s = s + src[1:I + 1, 2:J + 2]
                s = s + src[1:I + 1, 1:J + 1]
                dst[1:I + 1, 1:J + 1] = _cdiv(s, 5)
    return out


@pytest.mark.parametrize("family", ["reverse", "transpose", "addition", "matvec", "matmul", "jacobi", "jacobi2d"])
def test_random_binary64_bit_exact(cuda, family):
    from paper_1801_04348_b200 import last_run, programs, run_program

    rng = np.random.default_rng(0x64F + 131 * sum(map(ord, family)) + 7919 * SEED)
    kind = programs.original(family)
    for _ in range(DRAWS):
        P = _params(family, rng)
        shapes = programs.array_shapes(kind, P)
        arr = {k: _values(rng, s) for k, s in shapes.items()}
        with np.errstate(all="ignore"):
            want = _restate(family, P, arr)
        got = run_program(kind.text, P, {k: v.copy() for k, v in arr.items()})
        assert last_run().launch["dtype"] == "f64"
        for k in programs.FAMILIES[family].written:
            g, w = np.asarray(got[k]).reshape(-1), want[k].reshape(-1)
            nan = np.isnan(w)
            assert np.array_equal(np.isnan(g), nan), (family, P, k)
            assert np.array_equal(g[~nan].view(np.uint64), w[~nan].view(np.uint64)), (family, P, k)


def _restate_int(family, P, arr):
    """The programs on Python-int semantics for values whose results stay in
    int64 (numpy int64 arithmetic is then exact); Jacobi divides by C
    truncation (interp.py:43-46 on ints)."""
    out = {k: v.copy() for k, v in arr.items()}
    if family == "addition":
        N = P["N"]
        I, J, h = (N // P["B0"]) * P["B0"], min((N // (2 * P["B1"])) * P["B1"], N // 2), N // 2
        a, b, c = (x.reshape(N, N) for x in (arr["a"], arr["b"], out["c"]))
        c[:I, :J] = a[:I, :J] + b[:I, :J]
        c[:I, h:h + J] = a[:I, h:h + J] + b[:I, h:h + J]
    elif family == "matvec":
        N, t = P["N"], P["s"] * P["B"]
        R = (N // t) * t
        out["y"][:R] = arr["y"][:R] + arr["a"][:R] @ arr["x"]
    elif family == "matmul":
        n = P["n"]
        M = K = (n // P["B0"]) * P["B0"]
        Nc = (n // (P["ub1"] * P["s"])) * P["ub1"] * P["s"]
        out["c"][:M, :Nc] = arr["c"][:M, :Nc] + arr["a"][:M, :K] @ arr["b"][:K, :Nc]
    elif family == "jacobi":
        N, t = P["N"], P["s"] * P["B"]
        Pc = max(0, (N - 2) // t) * t
        a = out["a"]
        for step in range(P["T"]):
            src, dst = (a[N:], a[:N]) if step % 2 == 0 else (a[:N], a[N:])
            if Pc:
                s = src[0:Pc] + src[1:Pc + 1] + src[2:Pc + 2]
                dst[1:Pc + 1] = np.sign(s) * (np.abs(s) // 3)
    return out


@pytest.mark.parametrize("family", ["addition", "matvec", "matmul", "jacobi"])
def test_random_wide_int_exact(cuda, family):
    """ints whose results leave int32: the int64 kernels (never a wrapped
    int32 result), exact against int64 arithmetic."""
    from paper_1801_04348_b200 import last_run, marshal, programs, run_program

    rng = np.random.default_rng(0x164 + 17 * sum(map(ord, family)) + 7919 * SEED)
    kind = programs.original(family)
    lim = {"addition": 2**40, "matvec": 2**24, "matmul": 2**24, "jacobi": 2**50}[family]
    for _ in range(DRAWS):
        P = _params(family, rng)
        shapes = programs.array_shapes(kind, P)
        arr = {k: rng.integers(-lim, lim, size=s, dtype=np.int64) for k, s in shapes.items()}
        want = _restate_int(family, P, arr)
        got = run_program(kind.text, P, {k: v.copy() for k, v in arr.items()})
        srcs = {k: marshal.describe(k, v) for k, v in arr.items()}
        wide = family == "jacobi" or marshal.int_bound(family, P, srcs) > marshal.I32_MAX
        assert last_run().launch["dtype"] == ("i64" if wide else "i32"), (family, P)
        for k in programs.FAMILIES[family].written:
            assert np.array_equal(np.asarray(got[k]).reshape(-1), want[k].reshape(-1)), (family, P, k)
