"""Register-window Jacobi sweeps (csrc/k_jacobi_reg.cu), the default binding of
the staged leaf: one sweep through pk_jacobi_sweep over partial unit ranges,
every alignment of the two halves, narrow and 64-bit sums, against a torch
restatement of the step (jacobi.mfk / jacobi2d.mfk) and against the
shared-memory pipelines (PK_FLAG_GENERIC) -- bit-identical."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _launch(family, params, narrow, generic):
    from paper_1801_04348_b200 import _lib, binding, programs

    L = binding.make_launch(programs.original(family), params, (), _lib.DTYPE_I32)
    if narrow:
        L.flags |= _lib.FLAG_NARROW
    if generic:
        L.flags |= _lib.FLAG_GENERIC
    return L


def _sweep(torch, L, src, dst, lo, hi):
    from paper_1801_04348_b200 import _lib

    _lib.jacobi_sweep(L, src.data_ptr(), dst.data_ptr(), lo, hi, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()


def _want1d(torch, src, dst, lo, hi, P):
    out = dst.clone()
    a, b = max(lo, 1), min(hi, P + 1)
    if b > a:
        s = src[a - 1:b - 1].long() + src[a:b].long() + src[a + 1:b + 1].long()
        out[a:b] = torch.div(s, 3, rounding_mode="trunc").int()
    return out


@pytest.mark.parametrize("off_src", [0, 1, 2, 3])
@pytest.mark.parametrize("off_dst", [0, 1, 2, 3])
def test_jacobi1d_reg_every_alignment(cuda, off_src, off_dst):
    torch = cuda
    N = 70002 + off_src
    params = {"T": 1, "N": N, "s": 4, "B": 64}
    P = ((N - 2) // 256) * 256
    g = torch.Generator(device="cuda").manual_seed(off_src * 4 + off_dst)
    for narrow, lim in ((True, 1 << 20), (False, 2**31 - 1)):
        src_buf = torch.randint(-lim, lim, (N + 8,), dtype=torch.int32, device="cuda", generator=g)
        dst_buf = torch.randint(-lim, lim, (N + 8,), dtype=torch.int32, device="cuda", generator=g)
        src, dst0 = src_buf[off_src:off_src + N], dst_buf[off_dst:off_dst + N]
        for lo, hi in ((1, P + 1), (1, 5), (3, 1027), (517, 40001), (P - 9, P + 1), (P + 1, P + 1)):
            want = _want1d(torch, src, dst0, lo, hi, P)
            for generic in (False, True):
                buf = dst_buf.clone()
                dst = buf[off_dst:off_dst + N]
                _sweep(torch, _launch("jacobi", params, narrow, generic), src, dst, lo, hi)
                assert torch.equal(dst, want), (narrow, lo, hi, generic)
                assert torch.equal(buf[:off_dst], dst_buf[:off_dst]) and torch.equal(
                    buf[off_dst + N:], dst_buf[off_dst + N:])  # nothing outside the half


def _want2d(torch, src, dst, lo, hi, I, J):
    out = dst.clone()
    a, b = max(lo, 1), min(hi, I + 1)
    if b > a and J > 0:
        s = (src[a - 1:b - 1, 1:J + 1].long() + src[a + 1:b + 1, 1:J + 1].long() + src[a:b, 0:J].long() +
             src[a:b, 2:J + 2].long() + src[a:b, 1:J + 1].long())
        out[a:b, 1:J + 1] = torch.div(s, 5, rounding_mode="trunc").int()
    return out


@pytest.mark.parametrize("N,s,B0,B1", [(1026, 4, 16, 16), (1028, 2, 8, 32), (514, 3, 8, 20), (515, 2, 4, 8),
                                       (130, 1, 16, 4), (6, 1, 2, 4)])
def test_jacobi2d_reg_ranges_and_layouts(cuda, N, s, B0, B1):
    """N = 2 mod 4 (rows alternate 16/8-byte alignment), N = 0 mod 4, odd N
    (not the register kernel's layout: falls back), J < N - 2 tails."""
    torch = cuda
    params = {"T": 1, "N": N, "s": s, "B0": B0, "B1": B1}
    I = ((N - 2) // B0) * B0
    J = ((N - 2) // (s * B1)) * s * B1
    g = torch.Generator(device="cuda").manual_seed(N)
    for narrow, lim in ((True, 1 << 20), (False, 2**31 - 1)):
        a = torch.randint(-lim, lim, (2 * N, N), dtype=torch.int32, device="cuda", generator=g)
        src, dst0 = a[:N], a[N:]
        for lo, hi in ((1, I + 1), (1, 2), (2, 7), (3, I + 1), (I // 2, I // 2 + 5), (I, I + 1)):
            want = _want2d(torch, src, dst0, lo, hi, I, J)
            for generic in (False, True):
                b = a.clone()
                _sweep(torch, _launch("jacobi2d", params, narrow, generic), b[:N], b[N:], lo, hi)
                assert torch.equal(b[N:], want), (narrow, lo, hi, generic)
                assert torch.equal(b[:N], src)


def test_jacobi2d_reg_misaligned_base_falls_back(cuda):
    """Halves not on 16-byte boundaries: the shared-memory pipeline takes the
    sweep, same results."""
    torch = cuda
    N = 258
    params = {"T": 1, "N": N, "s": 2, "B0": 8, "B1": 16}
    I = J = 256
    g = torch.Generator(device="cuda").manual_seed(3)
    buf = torch.randint(-(1 << 20), 1 << 20, (2 * N * N + 4,), dtype=torch.int32, device="cuda", generator=g)
    for off in (1, 2):
        a = buf[off:off + 2 * N * N].view(2 * N, N)
        want = _want2d(torch, a[:N], a[N:], 1, I + 1, I, J)
        b_buf = buf.clone()
        b = b_buf[off:off + 2 * N * N].view(2 * N, N)
        _sweep(torch, _launch("jacobi2d", params, True, False), b[:N], b[N:], 1, I + 1)
        assert torch.equal(b[N:], want)


@pytest.mark.parametrize("where", ["overwritten", "boundary"])
def test_range_check_covers_what_the_program_reads(cuda, oracle_mod, where):
    """The narrow (int32-sum) path is chosen from the values a run can read:
    the half step 0 reads and the never-written points of the other half.
    Huge values in points step 0 overwrites do not matter; huge values in a
    never-written boundary point force the 64-bit sums -- both bit-exact."""
    import numpy as np

    from paper_1801_04348_b200 import programs, run_program

    rng = np.random.default_rng(12)
    big = 2**31 - 1
    N = 2002
    p1 = {"T": 5, "N": N, "s": 4, "B": 50}
    a = rng.integers(-(1 << 20), 1 << 20, size=2 * N).astype(np.int32)
    if where == "overwritten":
        a[1:N - 1] = big  # lower half, positions 1 .. P: written by step 0 before any read
    else:
        a[0] = big  # lower half, position 0: never written, read from step 1 on
        a[N - 1] = -big
    want = oracle_mod.run("jacobi", p1, {"a": a})["a"]
    got = run_program(programs.source("jacobi"), p1, {"a": a})["a"]
    assert np.array_equal(np.asarray(got).reshape(-1), np.asarray(want).reshape(-1))

    M = 130
    p2 = {"T": 4, "N": M, "s": 2, "B0": 8, "B1": 16}
    b = rng.integers(-(1 << 20), 1 << 20, size=(2 * M, M)).astype(np.int32)
    if where == "overwritten":
        b[M + 1:M + 129, 1:129] = big  # half 1, rows 1..I x cols 1..J
    else:
        b[M + 5, M - 1] = big  # half 1, column N-1 (> J): never written
        b[M + 7, 0] = -big
    want = oracle_mod.run("jacobi2d", p2, {"a": b})["a"]
    got = run_program(programs.source("jacobi2d"), p2, {"a": b})["a"]
    assert np.array_equal(np.asarray(got).reshape(-1), np.asarray(want).reshape(-1))
