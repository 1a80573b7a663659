"""GPU parity: the sm_100a kernels (through run_program -> ctypes -> libpk.so)
against the reference's own outputs and the CPU oracle.

Bars (BASELINE.json north_star):
* integer programs, reversal and transpose: bit-exact;
* float32 matmul: normalised error max|C_gpu - C_ref| / max_ij sum_k |a_ik b_kj|
  <= max(1e-5 * K / 1024, 2 * K * 2^-24)  (the second term covers tiny K, where
  a single fp32 rounding per step can exceed the K-scaled bound);
* float32 matvec (products split exactly and summed as a double-float pair
  on the GPU): within 2 fp32 ulps of the reference's binary64 result.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run(program, params, arrays, **kw):
    from paper_1801_04348_b200 import run_program

    return run_program(program, params, arrays, **kw)


def _text(v):
    from paper_1801_04348_b200 import programs

    return programs.source(v["family"]) if v["program"] == "original" else v["program"]


def _matmul_tol(K):
    return max(1e-5 * K / 1024.0, 2.0 * K * 2.0**-24)


def _check_float(family, params, inputs, got, want):
    w = np.asarray(want, dtype=np.float64)
    g = np.asarray(got, dtype=np.float64).reshape(w.shape)
    if family == "matmul":
        n = params["n"]
        a = np.asarray(inputs["a"], dtype=np.float64)
        b = np.asarray(inputs["b"], dtype=np.float64)
        scale = (np.abs(a) @ np.abs(b)).max() if n else 0.0
        scale = max(scale, np.abs(w).max() if w.size else 0.0, 1e-30)
        K = max(1, (n // params["B0"]) * params["B0"])
        assert np.abs(g - w).max() / scale <= _matmul_tol(K)
    else:
        tol = 2.0 * 2.0**-24 * np.abs(w) + 1e-30
        assert np.all(np.abs(g - w) <= tol)


def test_golden_vectors(cuda, golden):
    """Every reference-generated vector, original and case programs."""
    checked = 0
    for v in golden:
        if "error" in v:
            if v["error"] == "ZeroDivisionError":
                with pytest.raises(ZeroDivisionError):
                    _run(_text(v), v["params"], None)
            continue
        got = _run(_text(v), v["params"], v["inputs"])
        for name, want in v["outputs"].items():
            # Python floats run in binary64 with the interpreter's rounding
            # sequence (PK_DTYPE_F64): equal, not merely within tolerance
            assert got[name] == want, (v["family"], v["program"][:20], v["params"], name)
            if v["floats"] and name in ("c", "y"):
                _check_float(v["family"], v["params"], v["inputs"], got[name], want)
        checked += 1
    assert checked >= 100


FAMILY_CASES = {
    # family: (params, integer input range)
    "reverse": ({"N": 1 << 16, "s": 4, "B": 128}, 1 << 30),
    "transpose": ({"N": 256, "s": 4, "B0": 32, "B1": 8}, 1 << 30),
    "jacobi": ({"T": 7, "N": (1 << 14) + 2, "s": 4, "B": 64}, 1 << 30),
    "jacobi2d": ({"T": 5, "N": 130, "s": 2, "B0": 8, "B1": 16}, 1 << 30),
    "matvec": ({"N": 256, "s": 2, "B": 32}, 1 << 10),
    "matmul": ({"n": 128, "B0": 16, "ub1": 4, "s": 2}, 1 << 6),
    "addition": ({"N": 128, "B0": 8, "B1": 16}, 1 << 30),
}


def _random_inputs(family, params, lim, rng):
    from paper_1801_04348_b200 import programs

    kind = programs.original(family)
    shapes = programs.array_shapes(kind, params)
    return {k: rng.integers(-lim, lim, size=s, dtype=np.int64).astype(np.int32) for k, s in shapes.items()}


@pytest.mark.parametrize("family", sorted(FAMILY_CASES))
def test_every_leaf_matches_oracle(cuda, oracle_mod, family):
    """Force each case of the b200 table (staged / direct / granularity
    leaves) plus the generic thread mapping: all bit-identical to the oracle."""
    from paper_1801_04348_b200 import case_table, programs

    params, lim = FAMILY_CASES[family]
    rng = np.random.default_rng(0x1801)
    inputs = _random_inputs(family, params, lim, rng)
    want = oracle_mod.run(family, params, inputs)
    text = programs.source(family)
    for case in case_table(family, "b200").cases:
        for generic in (False, True):
            got = _run(text, params, inputs, case=case.index, generic=generic)
            for name in want:
                assert np.array_equal(np.asarray(got[name]).reshape(-1), np.asarray(want[name]).reshape(-1)), \
                    (family, case.index, generic, name)


def test_case_selected_on_live_machine(cuda):
    from paper_1801_04348_b200 import live_machine, select_case

    mv = live_machine()
    assert mv.values["T_B"] == 1024 and mv.values["R_B"] == 255
    assert mv.values["Z_B"] * 4 == mv.props["smem_per_block_optin"]
    # matvec caches x (N words) only if N <= Z_B: opt-in 227 KB keeps it at
    # N = 32768, the 48 KB static limit (== Fermi's 12288 words) does not
    assert select_case("matvec", {"N": 32768, "s": 1, "B": 256}, mv).applied == ()
    static = live_machine(smem="static")
    assert static.values["Z_B"] == 12288
    assert select_case("matvec", {"N": 32768, "s": 1, "B": 256}, static).applied == ("granularity", "caching-off")


def test_reversal_full_size_property(cuda):
    """BASELINE configs[4] at its size: 2^30 int32 words (4 GiB per array,
    byte offsets past 2^32).  One reversal equals torch.flip; reversing twice
    is the identity."""
    torch = cuda
    from paper_1801_04348_b200 import programs

    N = 1 << 30
    a = torch.randint(-(2**31), 2**31 - 1, (N,), dtype=torch.int32, device="cuda")
    out = _run(programs.source("reverse"), {"N": N, "s": 16, "B": 256}, {"a": a})
    assert torch.equal(out["c"], torch.flip(a, [0]))
    back = _run(programs.source("reverse"), {"N": N, "s": 16, "B": 256}, {"a": out["c"]})
    assert torch.equal(back["c"], a)


def test_transpose_full_size_property(cuda):
    """BASELINE configs[4] at its size: 32768^2 fp32 words (4 GiB per array)."""
    torch = cuda
    from paper_1801_04348_b200 import programs

    N = 32768
    a = torch.empty((N, N), dtype=torch.float32, device="cuda").uniform_(-1, 1)
    out = _run(programs.source("transpose"), {"N": N, "s": 8, "B0": 64, "B1": 8}, {"a": a})
    assert out["c"].dtype == torch.float32
    assert torch.equal(out["c"].reshape(N, N).view(torch.int32), a.t().view(torch.int32))


def _fp32_matmul_full_size(torch, tf32x3: bool, s: int = 16):
    from paper_1801_04348_b200 import last_run, programs

    n = 8192
    g = torch.Generator(device="cuda").manual_seed(0x1801)
    a, b, c = (torch.rand((n, n), device="cuda", generator=g) * 2 - 1 for _ in range(3))
    params = {"n": n, "B0": 128, "ub1": 8, "s": s}
    got = _run(programs.source("matmul"), params, {"a": a, "b": b, "c": c}, tf32x3=tf32x3)["c"]
    assert last_run().launch["dtype"] == "f32"
    want = c.double() + a.double() @ b.double()  # binary64 reference (the interpreter sums binary64)
    scale = (a.double().abs() @ b.double().abs()).max()
    err = ((got.double() - want).abs().max() / scale).item()
    return err


@pytest.mark.parametrize("s", [16, 8])
def test_matmul_fp32_full_size_tolerance(cuda, s):
    """BASELINE configs[1] headline at its size: n = 8192 on U[-1,1) against a
    binary64 product, normalised error <= 1e-5 * K / 1024 (north_star), on
    the 128 x 128 tile (s = 16) and the 128 x 64 producer-warp tile the
    bench's tuner picks (s = 8)."""
    err = _fp32_matmul_full_size(cuda, False, s)
    assert err <= _matmul_tol(8192), err


def test_matmul_tf32x3_full_size_tolerance(cuda):
    """The optional 3xTF32 tcgen05 variant at n = 8192, same bar."""
    err = _fp32_matmul_full_size(cuda, True)
    assert err <= _matmul_tol(8192), err


def test_matmul_fp32_tolerance_tuned_tile(cuda, oracle_mod):
    """n = 1024 with the tuned 128 x 128 tile vs the binary64 oracle."""
    from paper_1801_04348_b200 import last_run, programs

    n = 1024
    rng = np.random.default_rng(7)
    a = rng.uniform(-1, 1, (n, n)).astype(np.float32)
    b = rng.uniform(-1, 1, (n, n)).astype(np.float32)
    c = rng.uniform(-1, 1, (n, n)).astype(np.float32)
    params = {"n": n, "B0": 128, "ub1": 8, "s": 16}
    got = _run(programs.source("matmul"), params, {"a": a, "b": b, "c": c})
    assert last_run().applied == ()
    want = oracle_mod.run("matmul", params, {"a": a, "b": b, "c": c})["c"]
    scale = (np.abs(a.astype(np.float64)) @ np.abs(b.astype(np.float64))).max()
    err = np.abs(got["c"].astype(np.float64) - want).max() / scale
    assert err <= _matmul_tol(n), err


def test_matmul_integer_valued_fp32_is_exact(cuda, oracle_mod):
    """Integer-valued fp32 in [-8, 8]: every partial sum is an integer below
    2^24, so the fp32 result must equal the binary64 reference exactly."""
    from paper_1801_04348_b200 import programs

    n = 512
    rng = np.random.default_rng(11)
    a = rng.integers(-8, 9, (n, n)).astype(np.float32)
    b = rng.integers(-8, 9, (n, n)).astype(np.float32)
    for params in ({"n": n, "B0": 128, "ub1": 8, "s": 16}, {"n": n, "B0": 8, "ub1": 16, "s": 4}):
        got = _run(programs.source("matmul"), params, {"a": a, "b": b})
        want = oracle_mod.run("matmul", params, {"a": a, "b": b})["c"]
        assert np.array_equal(got["c"].astype(np.float64), want)


def test_tuned_and_generic_matmul_bit_identical(cuda):
    """Same ascending-k FFMA chain in both kernels: identical bits."""
    from paper_1801_04348_b200 import programs

    n = 256
    rng = np.random.default_rng(5)
    arrays = {k: rng.standard_normal((n, n)).astype(np.float32) for k in "abc"}
    # 64 x 64 register-blocked tile; 128 x 128 and 128 x 64 TMA-fed tiles (packed f32x2 FMAs)
    for params in ({"n": n, "B0": 64, "ub1": 8, "s": 8}, {"n": n, "B0": 128, "ub1": 8, "s": 16},
                   {"n": n, "B0": 128, "ub1": 8, "s": 8}):
        t = _run(programs.source("matmul"), params, arrays)["c"]
        g = _run(programs.source("matmul"), params, arrays, generic=True)["c"]
        assert np.array_equal(t.view(np.uint32), g.view(np.uint32)), params


def test_errors_mirror_reference(cuda):
    from paper_1801_04348_b200 import programs

    text = programs.source("jacobi")
    with pytest.raises(KeyError):
        _run(text, {"T": 1, "N": 10, "s": 1}, None)  # interp.py:75
    with pytest.raises(ZeroDivisionError):
        _run(text, {"T": 1, "N": 10, "s": 0, "B": 4}, None)
    with pytest.raises(NotImplementedError):
        _run(text, {"T": 1, "N": 10, "s": 1, "B": 4}, None, tracer=lambda *a: None)
    # a program outside the seven families runs on the generic path (generic.py)
    with pytest.warns(RuntimeWarning):
        out = _run("int N; int a[N]; meta_schedule { meta_for (int i = 0; i < N; i++) { a[i] = i; } }", {"N": 4}, None)
    assert out["a"] == [0, 1, 2, 3]


def test_inputs_not_mutated_and_missing_arrays_zero(cuda):
    from paper_1801_04348_b200 import programs

    a = list(range(16))
    keep = list(a)
    out = _run(programs.source("reverse"), {"N": 16, "s": 1, "B": 4}, {"a": a})
    assert a == keep  # interp.py:76-78 deep copies
    assert out["c"] == keep[::-1]
    out = _run(programs.source("reverse"), {"N": 16, "s": 1, "B": 4}, None)
    assert out["a"] == [0] * 16 and out["c"] == [0] * 16


def test_matmul_tf32x3_tcgen05_within_tolerance(cuda, oracle_mod):
    """Optional 3xTF32 tensor-core variant (reported separately): fp32-level
    accuracy against the binary64 oracle, same tolerance as the FFMA path."""
    from paper_1801_04348_b200 import programs

    for n in (256, 1024):
        rng = np.random.default_rng(n + 3)
        a = rng.uniform(-1, 1, (n, n)).astype(np.float32)
        b = rng.uniform(-1, 1, (n, n)).astype(np.float32)
        c = rng.uniform(-1, 1, (n, n)).astype(np.float32)
        params = {"n": n, "B0": 128, "ub1": 8, "s": 16}
        got = _run(programs.source("matmul"), params, {"a": a, "b": b, "c": c}, tf32x3=True)["c"]
        want = oracle_mod.run("matmul", params, {"a": a, "b": b, "c": c})["c"]
        scale = (np.abs(a.astype(np.float64)) @ np.abs(b.astype(np.float64))).max()
        err = np.abs(got.astype(np.float64) - want).max() / scale
        assert err <= _matmul_tol(n), (n, err)


# ---- BASELINE-size parity through properties that do not need the CPU oracle ----


@pytest.mark.parametrize("s", [16, 8])
def test_matmul_full_size_integer_valued_exact(cuda, s):
    """n = 8192 (BASELINE configs[1]) on the tuned TMA tile: integer-valued fp32
    in [-8, 8] keeps every partial sum an integer below 2^24, so the result
    must equal an exact binary64 product (torch float64 on the GPU)."""
    torch = cuda
    from paper_1801_04348_b200 import last_run, programs

    n = 8192
    g = torch.Generator(device="cuda").manual_seed(17)
    a = torch.randint(-8, 9, (n, n), device="cuda", generator=g).float()
    b = torch.randint(-8, 9, (n, n), device="cuda", generator=g).float()
    c = torch.randint(-8, 9, (n, n), device="cuda", generator=g).float()
    want = c.double() + a.double() @ b.double()
    # several launches: a missing proxy fence between the consumers' shared
    # loads and the next TMA refill once corrupted one tile every few runs
    for rep in range(4):
        got = _run(programs.source("matmul"), {"n": n, "B0": 128, "ub1": 8, "s": s},
                   {"a": a, "b": b, "c": c})["c"]
        assert last_run().applied == ()
        assert torch.equal(got.reshape(n, n).double(), want), rep


def _jacobi1d_torch(a, N, T, P):
    """Restatement of jacobi.mfk on the GPU (int64 sums, truncating division)."""
    torch = __import__("torch")
    h = [a[:N].long(), a[N:2 * N].long()]
    for t in range(T):
        src, dst = (h[1], h[0]) if t % 2 == 0 else (h[0], h[1])
        s = src[0:P] + src[1:P + 1] + src[2:P + 2]
        dst[1:P + 1] = torch.div(s, 3, rounding_mode="trunc")
    return torch.cat(h).int()


def test_jacobi1d_full_size_against_torch_restatement(cuda):
    """N = 2^28 + 2 (BASELINE configs[2]), 4 steps, full-range int32 inputs
    (64-bit sums) and narrow inputs (32-bit sums)."""
    torch = cuda
    from paper_1801_04348_b200 import programs

    N, T = (1 << 28) + 2, 4
    params = {"T": T, "N": N, "s": 16, "B": 256}
    P = ((N - 2) // (16 * 256)) * 16 * 256
    for lo, hi in ((-(2**31), 2**31 - 1), (-(1 << 20), 1 << 20)):
        a = torch.randint(lo, hi, (2 * N,), dtype=torch.int32, device="cuda")
        want = _jacobi1d_torch(a, N, T, P)
        got = _run(programs.source("jacobi"), params, {"a": a})["a"]
        assert torch.equal(got.reshape(-1), want)
        del a, want, got
        torch.cuda.empty_cache()


def test_jacobi2d_full_size_against_torch_restatement(cuda):
    """N = 16386 (BASELINE configs[3]), 3 steps, against a GPU restatement of
    jacobi2d.mfk (int64 sums, truncating division)."""
    torch = cuda
    from paper_1801_04348_b200 import programs

    N, T = 16386, 3
    params = {"T": T, "N": N, "s": 32, "B0": 64, "B1": 4}
    I = ((N - 2) // 64) * 64
    J = ((N - 2) // (32 * 4)) * 32 * 4
    a = torch.randint(-(1 << 20), 1 << 20, (2 * N, N), dtype=torch.int32, device="cuda")
    h = [a[:N].long(), a[N:].long()]
    for t in range(T):
        src, dst = (h[0], h[1]) if t % 2 == 0 else (h[1], h[0])
        s = (src[0:I, 1:J + 1] + src[2:I + 2, 1:J + 1] + src[1:I + 1, 0:J] + src[1:I + 1, 2:J + 2] +
             src[1:I + 1, 1:J + 1])
        dst[1:I + 1, 1:J + 1] = torch.div(s, 5, rounding_mode="trunc")
    want = torch.cat(h).int()
    del h
    got = _run(programs.source("jacobi2d"), params, {"a": a})["a"]
    assert torch.equal(got.reshape(2 * N, N), want)


def test_matvec_full_size_exact(cuda):
    """N = 32768 mat-vec on small integers: the int32 result equals an exact
    binary64 product."""
    torch = cuda
    from paper_1801_04348_b200 import programs

    N = 32768
    g = torch.Generator(device="cuda").manual_seed(3)
    a = torch.randint(-50, 50, (N, N), dtype=torch.int32, device="cuda", generator=g)
    x = torch.randint(-50, 50, (N,), dtype=torch.int32, device="cuda", generator=g)
    y = torch.randint(-50, 50, (N,), dtype=torch.int32, device="cuda", generator=g)
    got = _run(programs.source("matvec"), {"N": N, "s": 1, "B": 256}, {"a": a, "x": x, "y": y})["y"]
    want = (y.double() + a.double() @ x.double()).int()
    assert torch.equal(got.reshape(-1), want)


@pytest.mark.parametrize("rows", [(0, 640), (0, 1024), (1280, 2560), (4096, 8192)])
def test_matmul_split_schedule_exact_on_row_shares(cuda, rows):
    """Row shares whose tile count leaves a part-empty last wave take the
    order-preserving persistent split (k_matmul_tma_sched: a cut tile's second
    part waits for the first's c); integer-valued fp32 keeps every partial sum
    exact, so the rows must equal a binary64 product and the other rows stay
    untouched."""
    torch = cuda
    from paper_1801_04348_b200 import _lib, binding, programs

    n = 8192
    lo, hi = rows
    g = torch.Generator(device="cuda").manual_seed(lo + hi)
    a = torch.randint(-8, 9, (n, n), device="cuda", generator=g).float()
    b = torch.randint(-8, 9, (n, n), device="cuda", generator=g).float()
    c = torch.randint(-8, 9, (n, n), device="cuda", generator=g).float()
    want = c[lo:hi].double() + a[lo:hi].double() @ b.double()
    L = binding.make_launch(programs.original("matmul"), {"n": n, "B0": 128, "ub1": 8, "s": 16}, (),
                            _lib.DTYPE_F32, lo=lo, hi=hi)
    got = c.clone()
    _lib.launch(L, [a.data_ptr(), b.data_ptr(), got.data_ptr()], torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert torch.equal(got[lo:hi].double(), want)
    assert torch.equal(got[:lo], c[:lo]) and torch.equal(got[hi:], c[hi:])


@pytest.mark.parametrize("rows", [(0, 2048), (0, 1024), (512, 1920)])
def test_matmul_mid_tile_split_bit_identical(cuda, rows):
    """n = 2048 on the 128 x 64 TMA tile (3 CTAs per SM): 512 tiles for 444
    slots take the order-preserving split with every tile cut; random fp32 in
    [-1, 1): the bits must equal the 128 x 128 tile's and the generic kernel's
    (one ascending-k fma chain per output), rows outside the share untouched."""
    torch = cuda
    from paper_1801_04348_b200 import _lib, binding, programs

    n = 2048
    lo, hi = rows
    g = torch.Generator(device="cuda").manual_seed(hi)
    a, b, c = (torch.rand(n * n, device="cuda", generator=g) * 2 - 1 for _ in range(3))
    st = torch.cuda.current_stream().cuda_stream
    outs = []
    for params, generic in (({"n": n, "B0": 128, "ub1": 8, "s": 8}, False),
                            ({"n": n, "B0": 128, "ub1": 8, "s": 16}, False),
                            ({"n": n, "B0": 128, "ub1": 8, "s": 16}, True)):
        L = binding.make_launch(programs.original("matmul"), params, (), _lib.DTYPE_F32, lo=lo, hi=hi,
                                generic=generic)
        for rep in range(3):  # repeated launches: the split's waits and refills race for real
            got = c.clone()
            _lib.launch(L, [a.data_ptr(), b.data_ptr(), got.data_ptr()], st)
            torch.cuda.synchronize()
            if outs:
                assert torch.equal(got.view(torch.int32), outs[0].view(torch.int32)), (params, generic, rep)
            else:
                outs.append(got)
    got = outs[0].view(n, n)
    want = c.view(n, n)[lo:hi].double() + a.view(n, n)[lo:hi].double() @ b.view(n, n).double()
    scale = (a.view(n, n)[lo:hi].double().abs() @ b.view(n, n).double().abs()).max()
    assert ((got[lo:hi].double() - want).abs().max() / scale).item() <= _matmul_tol(n)
    assert torch.equal(got[:lo], c.view(n, n)[:lo]) and torch.equal(got[hi:], c.view(n, n)[hi:])


@pytest.mark.parametrize("n,rows", [(2048, (0, 2048)), (4096, (1024, 3072))])
def test_matmul_tile_options_bit_identical(cuda, monkeypatch, n, rows):
    """The 128 x 128 tile at one CTA per SM with a producer warp (Big1P, chosen
    when the tiles fill one wave), at two CTAs per SM (Big), and the tiles that
    read a's rows as they lie (PK_MM_ROWA=1): one ascending-k fma chain per
    output, so the bits equal the 128 x 64 tile's on random fp32 data."""
    torch = cuda
    from paper_1801_04348_b200 import _lib, binding, programs

    lo, hi = rows
    g = torch.Generator(device="cuda").manual_seed(n)
    a, b, c = (torch.rand(n * n, device="cuda", generator=g) * 2 - 1 for _ in range(3))
    st = torch.cuda.current_stream().cuda_stream
    ref = None
    for env, ub1 in (({}, 4), ({"PK_MM_TILE": "big1p"}, 8), ({"PK_MM_TILE": "big"}, 8),
                     ({"PK_MM_ROWA": "1"}, 8), ({"PK_MM_ROWA": "1"}, 4)):
        for k in ("PK_MM_TILE", "PK_MM_ROWA"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        L = binding.make_launch(programs.original("matmul"), {"n": n, "B0": 128, "ub1": ub1, "s": 16}, (),
                                _lib.DTYPE_F32, lo=lo, hi=hi)
        got = c.clone()
        _lib.launch(L, [a.data_ptr(), b.data_ptr(), got.data_ptr()], st)
        torch.cuda.synchronize()
        if ref is None:
            ref = got
        else:
            assert torch.equal(got.view(torch.int32), ref.view(torch.int32)), env
    assert torch.equal(ref[: lo * n], c[: lo * n]) and torch.equal(ref[hi * n:], c[hi * n:])


@pytest.mark.parametrize("N,scale", [(32768, 1.0), (4099, 1e30), (777, 1e-30)])
def test_matvec_float32_double_float_accumulation(cuda, N, scale):
    """float32 mat-vec at full size and at extreme magnitudes: the GPU's
    double-float sum rounded to float32 stays within 2 ulps of a binary64
    reference (the reference interpreter sums Python floats, binary64),
    with an absolute allowance of 2^-40 * sum|a*x| for rows that cancel."""
    torch = cuda
    from paper_1801_04348_b200 import programs

    g = torch.Generator(device="cuda").manual_seed(N)
    a = ((torch.rand((N, N), device="cuda", generator=g) - 0.5) * scale).float()
    x = (torch.rand((N,), device="cuda", generator=g) - 0.5).float()
    y = ((torch.rand((N,), device="cuda", generator=g) - 0.5) * scale).float()
    B = 512
    got = _run(programs.source("matvec"), {"N": N, "s": 1, "B": B}, {"a": a, "x": x, "y": y})["y"].reshape(-1)
    R = (N // B) * B  # rows the program's grid covers (whole blocks); the rest keep y
    assert torch.equal(got[R:], y[R:])
    want = y[:R].double() + a[:R].double() @ x.double()
    mag = y[:R].double().abs() + a[:R].double().abs() @ x.double().abs()
    err = (got[:R].double() - want).abs()
    assert bool((err <= 2.0 * 2.0**-24 * want.abs() + 2.0**-40 * mag).all())


def test_surviving_leaves_on_live_device(cuda):
    """a7 on the device itself: the live values leave the register-starved
    leaves (R_B below the estimate) dead, and selection restricted to the
    survivors picks the same leaf as the full evaluation."""
    from paper_1801_04348_b200 import cases, live_machine

    mv = live_machine()
    alive = {f: [c.index for c in cases.surviving(f, mv)] for f in ("reverse", "matvec", "matmul", "jacobi")}
    assert alive == {"reverse": [1, 3], "matvec": [1, 3], "matmul": [1, 3, 4], "jacobi": [1, 4]}
    for P in ({"n": 8192, "B0": 128, "ub1": 8, "s": 16}, {"n": 512, "B0": 256, "ub1": 4, "s": 64}):
        full = cases.select("matmul", P, mv)
        assert cases.select("matmul", P, mv, among=set(alive["matmul"])).index == full.index
