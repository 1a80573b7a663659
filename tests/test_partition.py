"""The partitioner (paper_1801_04348_b200/partition.py).

CPU: unit ranges, the ghost-zone schedule with an in-process exchanger and a
world_size-2 gloo run (torch.distributed point-to-point, as NCCL runs it on
GPUs), each against the oracle on the whole problem.  The per-step sweep
here is a small torch restatement (test infrastructure); on GPUs the same
schedule drives pk_jacobi_sweep (tests/test_gpu_partition.py).
"""

import os

import numpy as np
import pytest
import torch

from paper_1801_04348_b200 import partition


def cpu_sweep(family, P):
    N = P["N"]
    if family == "jacobi":
        def sweep(src, dst, lo, hi):
            if hi <= lo:
                return
            s = src.to(torch.int64)
            dst[lo:hi] = torch.div(s[lo - 1:hi - 1] + s[lo:hi] + s[lo + 1:hi + 1], 3,
                                   rounding_mode="trunc").to(torch.int32)
        return sweep
    J = max(0, (N - 2) // (P["s"] * P["B1"])) * P["s"] * P["B1"]

    def sweep2(src, dst, lo, hi):
        if hi <= lo or J <= 0:
            return
        s = src.view(N, N).to(torch.int64)
        d = dst.view(N, N)
        tot = (s[lo - 1:hi - 1, 1:J + 1] + s[lo + 1:hi + 1, 1:J + 1] + s[lo:hi, 0:J] +
               s[lo:hi, 2:J + 2] + s[lo:hi, 1:J + 1])
        d[lo:hi, 1:J + 1] = torch.div(tot, 5, rounding_mode="trunc").to(torch.int32)
    return sweep2


CASES = [
    ("jacobi", {"T": 9, "N": 130, "s": 2, "B": 8}),
    ("jacobi", {"T": 5, "N": 67, "s": 1, "B": 4}),  # tail: (N-2) % (s*B) != 0
    ("jacobi2d", {"T": 6, "N": 34, "s": 2, "B0": 4, "B1": 4}),
    ("jacobi2d", {"T": 3, "N": 21, "s": 1, "B0": 2, "B1": 3}),
]


def _initial(family, P, seed=3):
    rng = np.random.default_rng(seed)
    N = P["N"]
    size = 2 * N if family == "jacobi" else 2 * N * N
    return rng.integers(-(1 << 20), 1 << 20, size=size).astype(np.int32)


def _own(family, P, lo, hi, buf):
    """(index, values) of this rank's units in both halves."""
    N = P["N"]
    row = 1 if family == "jacobi" else N
    half = N * row
    idx = np.concatenate([np.arange(lo * row, hi * row), half + np.arange(lo * row, hi * row)])
    return idx, buf[idx]


@pytest.mark.parametrize("family", ["reverse", "transpose", "matvec", "matmul", "addition", "jacobi", "jacobi2d"])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_split_tiles_units_exactly(family, world):
    P = {"reverse": {"N": 1 << 12, "s": 4, "B": 32}, "transpose": {"N": 256, "s": 2, "B0": 32, "B1": 8},
         "matvec": {"N": 512, "s": 2, "B": 32}, "matmul": {"n": 512, "B0": 64, "ub1": 8, "s": 8},
         "addition": {"N": 96, "B0": 4, "B1": 8}, "jacobi": {"T": 1, "N": 1026, "s": 4, "B": 64},
         "jacobi2d": {"T": 1, "N": 130, "s": 2, "B0": 8, "B1": 16}}[family]
    first, end, align = partition.units(family, P)
    ranges = [partition.split(family, P, r, world) for r in range(world)]
    assert ranges[0][0] == first and ranges[-1][1] == end
    for (l0, h0), (l1, h1) in zip(ranges, ranges[1:]):
        assert h0 == l1
    if (end - first) // align >= world:  # enough whole tiles: boundaries on tiles
        for lo, hi in ranges[:-1]:
            assert (lo - first) % align == 0 and (hi - first) % align == 0


@pytest.mark.parametrize("family,P", CASES)
@pytest.mark.parametrize("world", [1, 2, 3])
@pytest.mark.parametrize("width", [1, 3, 16])
def test_local_ranks_match_oracle(oracle_mod, family, P, world, width):
    init = _initial(family, P)
    want = oracle_mod.run(family, P, {"a": init.reshape((-1,) if family == "jacobi" else (2 * P["N"], P["N"]))})["a"]
    want = np.asarray(want).reshape(-1)
    box = {}
    bufs = [torch.from_numpy(init.copy()) for _ in range(world)]
    exs = [partition.LocalExchanger(r, world, box) for r in range(world)]
    sweep = cpu_sweep(family, P)
    gens = [partition.run_stencil(family, P, bufs[r], exs[r], sweep, width=width) for r in range(world)]
    partition.drive_local(gens)
    got = init.copy()
    for r in range(world):
        lo, hi = partition.split(family, P, r, world)
        idx, vals = _own(family, P, lo, hi, bufs[r].numpy())
        got[idx] = vals
    assert np.array_equal(got, want)


def _gloo_worker(rank, world, port, family, P, width, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    init = _initial(family, P)
    buf = torch.from_numpy(init.copy())
    ex = partition.TorchExchanger()
    partition.drive(partition.run_stencil(family, P, buf, ex, cpu_sweep(family, P), width=width))
    lo, hi = partition.split(family, P, rank, world)
    idx, vals = _own(family, P, lo, hi, buf.numpy())
    gathered = [None] * world
    dist.all_gather_object(gathered, (idx, vals))
    if rank == 0:
        got = init.copy()
        for i, v in gathered:
            got[i] = v
        np.save(out_path, got)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("family,P", CASES[:1] + CASES[2:3])
def test_gloo_world2_matches_oracle(tmp_path, oracle_mod, family, P):
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = str(tmp_path / "got.npy")
    mp.spawn(_gloo_worker, args=(2, port, family, P, 4, out), nprocs=2, join=True)
    init = _initial(family, P)
    want = oracle_mod.run(family, P, {"a": init.reshape((-1,) if family == "jacobi" else (2 * P["N"], P["N"]))})["a"]
    assert np.array_equal(np.load(out), np.asarray(want).reshape(-1))


# ---- row-sharded families: run_rows over gloo (broadcast / scatter / gather) ----

ROW_CASES = [
    ("reverse", {"N": 1000, "s": 4, "B": 16}),               # tail: N % (s*B) != 0
    ("transpose", {"N": 40, "s": 2, "B0": 8, "B1": 4}),
    ("matvec", {"N": 48, "s": 2, "B": 8}),
    ("matmul", {"n": 40, "B0": 8, "ub1": 2, "s": 2}),        # row tail: 40 % 8 == 0, col tail 40 % 4 == 0
    ("matmul", {"n": 36, "B0": 8, "ub1": 2, "s": 4}),        # uncovered rows 32..35 and columns
    ("addition", {"N": 24, "B0": 4, "B1": 8}),
]


def _row_inputs(family, P, seed=5):
    from paper_1801_04348_b200 import programs

    shapes = programs.array_shapes(programs.original(family), P)
    rng = np.random.default_rng(seed)
    return {k: rng.integers(-50, 50, size=int(np.prod(s))).astype(np.int32) for k, s in shapes.items()}


def oracle_launch(oracle_mod, family, P, arrays):
    """CPU stand-in for pk_launch(lo, hi): the oracle's whole-program result,
    copied back only over the written shares of [lo, hi)."""
    from paper_1801_04348_b200 import programs

    shapes = programs.array_shapes(programs.original(family), P)

    def launch(lo, hi):
        host = {k: v.numpy().reshape(shapes[k]) for k, v in arrays.items()}
        res = oracle_mod.run(family, P, host)
        for name in programs.FAMILIES[family].written:
            off, cnt = partition.share_range(family, P, name, lo, hi)
            full = np.asarray(res[name]).reshape(-1)
            arrays[name][off:off + cnt] = torch.from_numpy(full[off:off + cnt].astype(np.int32))
    return launch


def _rows_worker(rank, world, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist

    from oracle import oracle as oracle_mod

    dist.init_process_group("gloo", rank=rank, world_size=world)
    for i, (family, P) in enumerate(ROW_CASES):
        init = _row_inputs(family, P)
        # only root holds the real inputs; the others start from garbage
        arrays = {k: torch.from_numpy(v.copy() if rank == 0 else np.full_like(v, 7777)) for k, v in init.items()}
        partition.run_rows(family, P, arrays, oracle_launch(oracle_mod, family, P, arrays))
        np.savez(out_path % (i, rank), **{k: v.numpy() for k, v in arrays.items()})
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_run_rows_gloo_every_rank_holds_the_oracle_result(tmp_path, oracle_mod, world):
    import socket

    import torch.multiprocessing as mp

    from paper_1801_04348_b200 import programs

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = str(tmp_path / "case%d_rank%d.npz")
    mp.spawn(_rows_worker, args=(world, port, out), nprocs=world, join=True)
    for i, (family, P) in enumerate(ROW_CASES):
        init = _row_inputs(family, P)
        shapes = programs.array_shapes(programs.original(family), P)
        want = oracle_mod.run(family, P, {k: v.reshape(shapes[k]) for k, v in init.items()})
        for r in range(world):
            got = np.load(out % (i, r))
            for name in programs.FAMILIES[family].written:
                assert np.array_equal(got[name], np.asarray(want[name]).reshape(-1)), (family, P, r, name)
            for name in partition.REPLICATED.get(family, ()):
                assert np.array_equal(got[name], init[name]), (family, r, name)


def test_share_range_rules():
    P = {"n": 256, "B0": 64, "ub1": 8, "s": 16}
    assert partition.share_range("matmul", P, "a", 64, 128) == (64 * 256, 64 * 256)
    assert partition.share_range("matmul", P, "b", 64, 128) == (0, 256 * 256)
    assert partition.share_range("reverse", {"N": 4096, "s": 4, "B": 64}, "c", 0, 1024) == (3072, 1024)
    assert partition.share_range("matvec", {"N": 64, "s": 1, "B": 8}, "y", 8, 16) == (8, 8)
    with pytest.raises(KeyError):
        partition.share_range("jacobi", {"T": 1, "N": 10, "s": 1, "B": 2}, "a", 1, 2)
