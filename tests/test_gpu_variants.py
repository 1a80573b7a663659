"""Optional variants reported beside the leaves: temporally blocked 1-D
Jacobi (bit-identical to the per-step program) and its half bookkeeping."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("h", [3, 7, 9])
@pytest.mark.parametrize("T", [0, 1, 2, 3, 4, 8, 11, 20])
def test_temporal_jacobi1d_matches_oracle(cuda, oracle_mod, h, T):
    from paper_1801_04348_b200 import programs, run_program

    rng = np.random.default_rng(T * 31 + h)
    for N, s, B in ((20002, 4, 64), (9001, 3, 100)):  # full coverage; tail + odd N
        params = {"T": T, "N": N, "s": s, "B": B}
        a = rng.integers(-(1 << 20), 1 << 20, size=2 * N).astype(np.int32)
        want = oracle_mod.run("jacobi", params, {"a": a})["a"]
        got = run_program(programs.source("jacobi"), params, {"a": a}, temporal=h)["a"]
        assert np.array_equal(np.asarray(got).reshape(-1), np.asarray(want).reshape(-1)), (T, h, N)


def test_temporal_jacobi1d_wide_values(cuda, oracle_mod):
    """Full-range int32 inputs force 64-bit sums inside the fused steps too."""
    from paper_1801_04348_b200 import programs, run_program

    rng = np.random.default_rng(4)
    params = {"T": 13, "N": 40002, "s": 8, "B": 128}
    a = rng.integers(-(2**31), 2**31 - 1, size=2 * params["N"]).astype(np.int32)
    want = oracle_mod.run("jacobi", params, {"a": a})["a"]
    got = run_program(programs.source("jacobi"), params, {"a": a}, temporal=5)["a"]
    assert np.array_equal(np.asarray(got).reshape(-1), np.asarray(want).reshape(-1))


def test_occupancy_model_on_live_device(cuda, oracle_mod):
    """The occupancy counter's register file is the live regsPerMultiprocessor
    and its warp slots the live resident-warp count; selection on that model
    drives the same kernels."""
    from paper_1801_04348_b200 import interp, machine, programs, run_program

    mv = machine.live(occupancy=1)
    assert mv.table == "b200-occ" and mv.values["R_F"] == mv.props["regs_per_sm"] == 65536
    assert machine.warp_slots(mv) == 64
    rng = np.random.default_rng(7)
    params = {"T": 5, "N": 8194, "s": 4, "B": 256}
    a = rng.integers(-1000, 1000, size=2 * params["N"]).astype(np.int32)
    want = oracle_mod.run("jacobi", params, {"a": a})["a"]
    got = run_program(programs.source("jacobi"), params, {"a": a}, machine=mv)["a"]
    assert np.array_equal(np.asarray(got).reshape(-1), np.asarray(want).reshape(-1))
    info = interp.last_run()
    assert info.case == 1 and not info.fallback


@pytest.mark.parametrize("h", [3, 5, 11])
@pytest.mark.parametrize("T", [0, 1, 2, 3, 4, 6, 9, 14])
def test_temporal_jacobi2d_matches_oracle(cuda, oracle_mod, h, T):
    """2-D temporal blocking: bit-identical to the per-step program, including
    uncovered tails (J < N-2, I < N-2), odd N and tiles cut by the edges."""
    from paper_1801_04348_b200 import programs, run_program

    rng = np.random.default_rng(T * 17 + h)
    for N, s, B0, B1 in ((258, 4, 8, 8), (301, 2, 4, 16), (130, 1, 16, 4)):
        params = {"T": T, "N": N, "s": s, "B0": B0, "B1": B1}
        a = rng.integers(-(1 << 20), 1 << 20, size=(2 * N, N)).astype(np.int32)
        want = oracle_mod.run("jacobi2d", params, {"a": a})["a"]
        got = run_program(programs.source("jacobi2d"), params, {"a": a}, temporal=h)["a"]
        assert np.array_equal(np.asarray(got).reshape(-1), np.asarray(want).reshape(-1)), (T, h, N)


def test_temporal_jacobi2d_wide_values(cuda, oracle_mod):
    """Full-range int32 inputs force 64-bit sums inside the fused steps."""
    from paper_1801_04348_b200 import programs, run_program

    rng = np.random.default_rng(21)
    params = {"T": 11, "N": 386, "s": 4, "B0": 8, "B1": 16}
    a = rng.integers(-(2**31), 2**31 - 1, size=(2 * 386, 386)).astype(np.int32)
    want = oracle_mod.run("jacobi2d", params, {"a": a})["a"]
    got = run_program(programs.source("jacobi2d"), params, {"a": a}, temporal=5)["a"]
    assert np.array_equal(np.asarray(got).reshape(-1), np.asarray(want).reshape(-1))


def test_temporal_jacobi1d_full_size_matches_per_step(cuda):
    """N = 2^28 + 2 (BASELINE configs[2]): the register-resident h = 15 passes
    and the per-step sweeps leave identical double buffers (T = 37: two
    15-step passes, a 5-step pass and the closing sweep)."""
    torch = cuda
    from paper_1801_04348_b200 import programs, run_program

    N = (1 << 28) + 2
    params = {"T": 37, "N": N, "s": 16, "B": 256}
    g = torch.Generator(device="cuda").manual_seed(99)
    a = torch.randint(-(1 << 20), 1 << 20, (2 * N,), dtype=torch.int32, device="cuda", generator=g)
    want = run_program(programs.source("jacobi"), params, {"a": a})["a"]
    got = run_program(programs.source("jacobi"), params, {"a": a}, temporal=15)["a"]
    assert torch.equal(got, want)


def test_temporal_jacobi2d_full_size_matches_per_step(cuda):
    """N = 16386 (BASELINE configs[3]): the register-wavefront h = 7 passes and
    the per-step sweeps leave identical double buffers (T = 17: two 7-step
    passes, a 1-step remainder and the closing sweep)."""
    torch = cuda
    from paper_1801_04348_b200 import programs, run_program

    N = 16386
    params = {"T": 17, "N": N, "s": 32, "B0": 64, "B1": 4}
    g = torch.Generator(device="cuda").manual_seed(98)
    a = torch.randint(-(1 << 20), 1 << 20, (2 * N, N), dtype=torch.int32, device="cuda", generator=g)
    want = run_program(programs.source("jacobi2d"), params, {"a": a})["a"]
    got = run_program(programs.source("jacobi2d"), params, {"a": a}, temporal=7)["a"]
    assert torch.equal(got, want)
