"""Randomised parity: many small parameter draws per family (tails, odd
extents, block sizes that are not warp multiples, every leaf), CUDA vs the
CPU oracle, bit-exact.  Seeds are fixed so failures reproduce; PK_FUZZ_DRAWS
and PK_FUZZ_SEED widen a run (long soak runs on the GPU box)."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _draw(family, rng):
    r = lambda lo, hi: int(rng.integers(lo, hi))  # noqa: E731
    if family == "reverse":
        return {"N": r(1, 5000), "s": r(1, 9), "B": r(1, 300)}
    if family == "transpose":
        return {"N": r(1, 300), "s": r(1, 5), "B0": r(1, 70), "B1": r(1, 40)}
    if family == "jacobi":
        return {"T": r(0, 7), "N": r(2, 6000), "s": r(1, 9), "B": r(1, 300)}
    if family == "jacobi2d":
        return {"T": r(0, 5), "N": r(3, 200), "s": r(1, 9), "B0": r(1, 40), "B1": r(1, 40)}
    if family == "matvec":
        return {"N": r(1, 300), "s": r(1, 5), "B": r(1, 300)}
    if family == "matmul":
        return {"n": r(1, 200), "B0": r(1, 40), "ub1": r(1, 20), "s": r(1, 9)}
    return {"N": r(1, 200), "B0": r(1, 40), "B1": r(1, 40)}


def _threads_ok(family, P):
    from paper_1801_04348_b200 import programs

    return programs.threads_per_block(family, P) <= 1024


@pytest.mark.parametrize("family", ["reverse", "transpose", "jacobi", "jacobi2d", "matvec", "matmul", "addition"])
def test_random_parameters_match_oracle(cuda, oracle_mod, family):
    from paper_1801_04348_b200 import case_table, programs, run_program

    rng = np.random.default_rng(0xF022 + sum(map(ord, family)) + 7919 * int(os.environ.get("PK_FUZZ_SEED", 0)))
    kind = programs.original(family)
    ncases = len(case_table(family, "b200").cases)
    done = 0
    while done < int(os.environ.get("PK_FUZZ_DRAWS", 25)):
        P = _draw(family, rng)
        if not _threads_ok(family, P):
            continue
        shapes = programs.array_shapes(kind, P)
        lim = 1 << 6 if family in ("matvec", "matmul") else 1 << 30
        arrays = {k: rng.integers(-lim, lim, size=s).astype(np.int32) for k, s in shapes.items()}
        want = oracle_mod.run(family, P, arrays)
        case = int(rng.integers(1, ncases + 1))
        generic = bool(rng.integers(0, 2))
        got = run_program(kind.text, P, arrays, case=case, generic=generic)
        for name in programs.FAMILIES[family].written:
            assert np.array_equal(np.asarray(got[name]).reshape(-1), np.asarray(want[name]).reshape(-1)), \
                (family, P, case, generic, name)
        done += 1


EMPTY = {
    "reverse": [{"N": 0, "s": 2, "B": 32}, {"N": 5, "s": 2, "B": 32}],
    "transpose": [{"N": 0, "s": 1, "B0": 4, "B1": 4}, {"N": 3, "s": 2, "B0": 4, "B1": 4}],
    "jacobi": [{"T": 3, "N": 2, "s": 1, "B": 4}, {"T": 0, "N": 50, "s": 1, "B": 4}, {"T": 2, "N": 5, "s": 2, "B": 4}],
    "jacobi2d": [{"T": 2, "N": 2, "s": 1, "B0": 2, "B1": 2}, {"T": 0, "N": 9, "s": 1, "B0": 2, "B1": 2}],
    "matvec": [{"N": 0, "s": 1, "B": 32}, {"N": 7, "s": 1, "B": 32}],
    "matmul": [{"n": 0, "B0": 4, "ub1": 2, "s": 2}, {"n": 3, "B0": 4, "ub1": 2, "s": 2}],
    "addition": [{"N": 0, "B0": 2, "B1": 2}, {"N": 3, "B0": 4, "B1": 4}],
}


@pytest.mark.parametrize("family", sorted(EMPTY))
def test_empty_arrays_and_no_covered_block(cuda, oracle_mod, family):
    """Zero-sized arrays, extents below one block (the grid covers nothing),
    T = 0 and stencils without interior: nothing is launched that could fail,
    and every array comes back as the reference leaves it."""
    from paper_1801_04348_b200 import programs, run_program

    kind = programs.original(family)
    rng = np.random.default_rng(5)
    for P in EMPTY[family]:
        shapes = programs.array_shapes(kind, P)
        arrays = {k: rng.integers(-100, 100, size=s).astype(np.int32) for k, s in shapes.items()}
        want = oracle_mod.run(family, P, arrays)
        got = run_program(kind.text, P, arrays)
        for name in shapes:
            assert np.array_equal(np.asarray(got[name]).reshape(-1), np.asarray(want[name]).reshape(-1)), (P, name)


@pytest.mark.parametrize("family", ["matvec", "matmul"])
def test_random_float32_within_tolerance(cuda, oracle_mod, family):
    """float32 draws for the accumulating families against the binary64
    oracle: matmul within max(1e-5*K/1024, 2*K*2^-24) of max sum|a||b|,
    mat-vec within 2 ulps (+2^-40 sum|a x| for cancelling rows)."""
    from paper_1801_04348_b200 import case_table, programs, run_program

    rng = np.random.default_rng(0xF1 + sum(map(ord, family)) + 7919 * int(os.environ.get("PK_FUZZ_SEED", 0)))
    kind = programs.original(family)
    ncases = len(case_table(family, "b200").cases)
    done = 0
    while done < int(os.environ.get("PK_FUZZ_DRAWS", 25)):
        P = _draw(family, rng)
        if not _threads_ok(family, P):
            continue
        shapes = programs.array_shapes(kind, P)
        arrays = {k: rng.uniform(-1, 1, size=s).astype(np.float32) for k, s in shapes.items()}
        want = np.asarray(oracle_mod.run(family, P, arrays)["y" if family == "matvec" else "c"], dtype=np.float64)
        case = int(rng.integers(1, ncases + 1))
        generic = bool(rng.integers(0, 2))
        got = run_program(kind.text, P, arrays, case=case, generic=generic)
        g = np.asarray(got["y" if family == "matvec" else "c"], dtype=np.float64).reshape(want.shape)
        if family == "matmul":
            a, b = arrays["a"].astype(np.float64), arrays["b"].astype(np.float64)
            scale = max((np.abs(a) @ np.abs(b)).max() if P["n"] else 0.0, 1e-30)
            K = max(1, P["n"])
            assert np.abs(g - want).max(initial=0.0) / scale <= max(1e-5 * K / 1024.0, 2.0 * K * 2.0**-24), \
                (P, case, generic)
        else:
            a, x = arrays["a"].astype(np.float64), arrays["x"].astype(np.float64)
            mag = np.abs(arrays["y"].astype(np.float64)) + np.abs(a) @ np.abs(x)
            assert np.all(np.abs(g - want) <= 2.0 * 2.0**-24 * np.abs(want) + 2.0**-40 * mag), (P, case, generic)
        done += 1


@pytest.mark.parametrize("family", ["jacobi", "jacobi2d"])
def test_random_temporal_blocking_matches_oracle(cuda, oracle_mod, family):
    """Temporally blocked stencils (register-resident 1-D, register wavefront
    2-D, and their shared-memory fallbacks for odd N) over random extents,
    step counts and block depths h, narrow and full-range values: bit-exact."""
    from paper_1801_04348_b200 import programs, run_program

    rng = np.random.default_rng(0x7E + sum(map(ord, family)) + 7919 * int(os.environ.get("PK_FUZZ_SEED", 0)))
    kind = programs.original(family)
    done = 0
    while done < int(os.environ.get("PK_FUZZ_DRAWS", 25)):
        P = _draw(family, rng)
        if family == "jacobi":
            P["N"] = int(rng.integers(2, 40000))
        else:
            P["N"] = int(rng.integers(3, 400))
        P["T"] = int(rng.integers(0, 40))
        if not _threads_ok(family, P):
            continue
        h = int(rng.integers(1, 17 if family == "jacobi" else 9))
        lim = 1 << 20 if rng.integers(0, 2) else 2**31 - 1
        shapes = programs.array_shapes(kind, P)
        arrays = {k: rng.integers(-lim, lim, size=s, dtype=np.int64).astype(np.int32) for k, s in shapes.items()}
        want = oracle_mod.run(family, P, arrays)["a"]
        got = run_program(kind.text, P, arrays, temporal=h)["a"]
        assert np.array_equal(np.asarray(got).reshape(-1), np.asarray(want).reshape(-1)), (P, h, lim)
        done += 1
