"""Partitioned execution on one GPU: every rank's unit range launched through
pk_launch(lo, hi) / pk_jacobi_sweep, ranks simulated in-process (the box has
one GPU; the same schedule runs one process per GPU over NCCL in bench.py)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _dev(torch, arr):
    return torch.from_numpy(np.ascontiguousarray(arr).reshape(-1)).cuda()


@pytest.mark.parametrize("family,params", [
    ("reverse", {"N": 1 << 16, "s": 4, "B": 64}),
    ("transpose", {"N": 512, "s": 4, "B0": 32, "B1": 8}),
    ("matvec", {"N": 512, "s": 2, "B": 64}),
    ("matmul", {"n": 512, "B0": 64, "ub1": 8, "s": 16}),
    ("addition", {"N": 256, "B0": 4, "B1": 64}),
])
@pytest.mark.parametrize("world", [2, 3, 8])
def test_row_shards_reassemble_full_run(cuda, family, params, world):
    torch = cuda
    from paper_1801_04348_b200 import _lib, binding, cases, partition, programs

    kind = programs.original(family)
    shapes = programs.array_shapes(kind, params)
    rng = np.random.default_rng(world)
    init = {k: rng.integers(-64, 64, size=s).astype(np.int32) for k, s in shapes.items()}
    sel = cases.select(kind, params, "nominal")
    full = [_dev(torch, init[a.name]) for a in programs.FAMILIES[family].arrays]
    _lib.launch(binding.make_launch(kind, params, sel.applied), [t.data_ptr() for t in full])
    shard = [_dev(torch, init[a.name]) for a in programs.FAMILIES[family].arrays]
    for r in range(world):
        lo, hi = partition.split(family, params, r, world)
        if hi > lo:
            L = binding.make_launch(kind, params, sel.applied, lo=lo, hi=hi)
            _lib.launch(L, [t.data_ptr() for t in shard])
    torch.cuda.synchronize()
    for f, s in zip(full, shard):
        assert torch.equal(f, s)


@pytest.mark.parametrize("family,params", [
    ("jacobi", {"T": 11, "N": (1 << 16) + 2, "s": 4, "B": 64}),
    ("jacobi", {"T": 5, "N": 1001, "s": 2, "B": 16}),  # tail and odd N (scalar path)
    ("jacobi2d", {"T": 7, "N": 258, "s": 2, "B0": 8, "B1": 16}),
    ("jacobi2d", {"T": 4, "N": 67, "s": 1, "B0": 4, "B1": 8}),
])
@pytest.mark.parametrize("world", [1, 2, 4])
def test_halo_exchange_ranks_match_oracle(cuda, oracle_mod, family, params, world):
    torch = cuda
    from paper_1801_04348_b200 import _lib, binding, cases, partition, programs

    kind = programs.original(family)
    N = params["N"]
    size = 2 * N if family == "jacobi" else 2 * N * N
    rng = np.random.default_rng(17)
    init = rng.integers(-(1 << 20), 1 << 20, size=size).astype(np.int32)
    want = np.asarray(oracle_mod.run(family, params, {"a": init.reshape((-1,) if family == "jacobi" else (2 * N, N))})["a"]).reshape(-1)
    sel = cases.select(kind, params, "nominal")
    L = binding.make_launch(kind, params, sel.applied)
    narrow = _lib.jacobi_narrow(L, _dev(torch, init).data_ptr())
    assert narrow
    L.flags |= _lib.FLAG_NARROW

    def sweep(src, dst, lo, hi):
        _lib.jacobi_sweep(L, src.data_ptr(), dst.data_ptr(), lo, hi,
                          torch.cuda.current_stream().cuda_stream)

    box = {}
    bufs = [_dev(torch, init) for _ in range(world)]
    exs = [partition.LocalExchanger(r, world, box) for r in range(world)]
    gens = [partition.run_stencil(family, params, bufs[r], exs[r], sweep, width=3) for r in range(world)]
    partition.drive_local(gens)
    torch.cuda.synchronize()
    got = init.copy()
    row = 1 if family == "jacobi" else N
    half = N * row
    for r in range(world):
        lo, hi = partition.split(family, params, r, world)
        b = bufs[r].cpu().numpy()
        for off in (0, half):
            got[off + lo * row: off + hi * row] = b[off + lo * row: off + hi * row]
    assert np.array_equal(got, want)


def test_wide_path_for_large_values(cuda, oracle_mod):
    """Values beyond the narrow bound force 64-bit sums; results stay exact."""
    from paper_1801_04348_b200 import programs, run_program

    N = 4098
    rng = np.random.default_rng(2)
    a = rng.integers(-(2**31), 2**31 - 1, size=2 * N).astype(np.int32)
    params = {"T": 6, "N": N, "s": 4, "B": 64}
    got = run_program(programs.source("jacobi"), params, {"a": a})["a"]
    want = oracle_mod.run("jacobi", params, {"a": a})["a"]
    assert np.array_equal(np.asarray(got).reshape(-1), np.asarray(want).reshape(-1))
    N2 = 66
    a2 = rng.integers(-(2**31), 2**31 - 1, size=(2 * N2, N2)).astype(np.int32)
    p2 = {"T": 4, "N": N2, "s": 2, "B0": 4, "B1": 8}
    got = run_program(programs.source("jacobi2d"), p2, {"a": a2})["a"]
    want = oracle_mod.run("jacobi2d", p2, {"a": a2})["a"]
    assert np.array_equal(np.asarray(got).reshape(-1), np.asarray(want).reshape(-1))


@pytest.mark.parametrize("family,params", [
    ("reverse", {"N": 1 << 12, "s": 4, "B": 64}),
    ("matmul", {"n": 256, "B0": 64, "ub1": 8, "s": 16}),
    ("matvec", {"N": 256, "s": 1, "B": 64}),
    ("transpose", {"N": 128, "s": 4, "B0": 32, "B1": 8}),
    ("addition", {"N": 64, "B0": 4, "B1": 16}),
])
def test_run_host_shares_reassemble_oracle(cuda, oracle_mod, family, params):
    """pk_run_host with a rank's unit range copies only that share; the
    shares of 3 ranks written into one host buffer equal the oracle."""
    from paper_1801_04348_b200 import _lib, binding, cases, partition, programs

    kind = programs.original(family)
    shapes = programs.array_shapes(kind, params)
    rng = np.random.default_rng(9)
    init = {k: rng.integers(-32, 32, size=s).astype(np.int32) for k, s in shapes.items()}
    want = oracle_mod.run(family, params, init)
    host = {k: np.ascontiguousarray(v.copy()) for k, v in init.items()}
    sel = cases.select(kind, params, "nominal")
    for r in range(3):
        lo, hi = partition.split(family, params, r, 3)
        L = binding.make_launch(kind, params, sel.applied, lo=lo, hi=hi)
        _lib.run_host(L, [host[a.name].ctypes.data for a in programs.FAMILIES[family].arrays], 0)
    for name in programs.FAMILIES[family].written:
        assert np.array_equal(host[name].reshape(-1), np.asarray(want[name]).reshape(-1)), name


@pytest.mark.parametrize("family,params,share", [
    ("matmul", {"n": 4096, "B0": 128, "ub1": 8, "s": 16}, None),
    ("matmul", {"n": 4096, "B0": 128, "ub1": 8, "s": 16}, (1000, 3001)),
    ("matmul", {"n": 8192, "B0": 128, "ub1": 8, "s": 16}, None),   # 8 chunks x 4 reduction slices
    ("matmul", {"n": 2048, "B0": 128, "ub1": 8, "s": 16}, None),   # fewer chunks than slices
    ("matmul", {"n": 8192, "B0": 128, "ub1": 8, "s": 16}, (256, 5888)),
    ("reverse", {"N": 1 << 25, "s": 16, "B": 256}, None),
    ("reverse", {"N": 1 << 25, "s": 16, "B": 256}, (12345, 30000000)),
    ("matvec", {"N": 8192, "s": 1, "B": 256}, None),
    ("transpose", {"N": 4096, "s": 8, "B0": 64, "B1": 8}, None),
    ("addition", {"N": 4096, "B0": 4, "B1": 64}, None),
])
def test_run_host_pipeline_matches_device_launch(cuda, family, params, share):
    """Large host-buffer runs are cut into row chunks whose PCIe traffic
    overlaps the kernels; the result equals one pk_launch on device buffers."""
    import torch

    from paper_1801_04348_b200 import _lib, binding, cases, programs

    kind = programs.original(family)
    shapes = programs.array_shapes(kind, params)
    f32 = family in ("matmul", "matvec")
    rng = np.random.default_rng(11)
    init = {}
    for k, s in shapes.items():
        if f32:
            init[k] = rng.uniform(-1, 1, size=s).astype(np.float32)
        else:
            init[k] = rng.integers(-1000, 1000, size=s).astype(np.int32)
    sel = cases.select(kind, params, "nominal")
    dtype = _lib.DTYPE_F32 if f32 else _lib.DTYPE_I32
    lo, hi = share if share else (0, 0)
    L = binding.make_launch(kind, params, sel.applied, dtype, lo=lo, hi=hi)
    names = [a.name for a in programs.FAMILIES[family].arrays]
    dev = [torch.from_numpy(init[n].reshape(-1).copy()).cuda() for n in names]
    _lib.launch(L, [t.data_ptr() for t in dev], torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    host = {n: np.ascontiguousarray(init[n].copy()) for n in names}
    _lib.run_host(L, [host[n].ctypes.data for n in names], 0)
    for n, t in zip(names, dev):
        if n in programs.FAMILIES[family].written:
            # outside a share both sides keep the initial contents
            want = t.cpu().numpy().reshape(-1)
            assert np.array_equal(host[n].reshape(-1).view(np.int32), want.view(np.int32)), n


@pytest.mark.parametrize("family,params", [
    ("matmul", {"n": 512, "B0": 128, "ub1": 8, "s": 16}),
    ("reverse", {"N": 1 << 16, "s": 16, "B": 256}),
    ("matvec", {"N": 1024, "s": 1, "B": 256}),
])
def test_run_rows_with_pk_launcher(cuda, oracle_mod, family, params):
    """run_rows' GPU launcher (pk_launch over the rank's unit range) in a
    one-rank process group, against the oracle."""
    import socket

    import torch
    import torch.distributed as dist

    from paper_1801_04348_b200 import partition, programs

    kind = programs.original(family)
    shapes = programs.array_shapes(kind, params)
    rng = np.random.default_rng(13)
    init = {k: rng.integers(-40, 40, size=s).astype(np.int32) for k, s in shapes.items()}
    want = oracle_mod.run(family, params, init)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    dist.init_process_group("gloo", init_method="tcp://127.0.0.1:%d" % port, rank=0, world_size=1)
    try:
        arrays = {k: torch.from_numpy(v.reshape(-1).copy()).cuda() for k, v in init.items()}
        partition.run_rows(family, params, arrays, partition.pk_launcher(family, params, arrays))
        torch.cuda.synchronize()
        for name in programs.FAMILIES[family].written:
            assert np.array_equal(arrays[name].cpu().numpy(), np.asarray(want[name]).reshape(-1)), name
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("family,params", [
    ("reverse", {"N": 100000, "s": 4, "B": 64}),
    ("transpose", {"N": 300, "s": 2, "B0": 16, "B1": 8}),
    ("matvec", {"N": 1000, "s": 1, "B": 64}),
    ("matmul", {"n": 512, "B0": 128, "ub1": 8, "s": 16}),
    ("matmul", {"n": 200, "B0": 16, "ub1": 4, "s": 2}),
    ("addition", {"N": 96, "B0": 4, "B1": 16}),
    ("jacobi", {"T": 37, "N": 20002, "s": 4, "B": 64}),
    ("jacobi", {"T": 9, "N": 1001, "s": 3, "B": 32}),
    ("jacobi2d", {"T": 21, "N": 130, "s": 2, "B0": 4, "B1": 8}),
    ("jacobi2d", {"T": 6, "N": 67, "s": 1, "B0": 2, "B1": 16}),
])
@pytest.mark.parametrize("ndev,halo", [(2, 0), (3, 0), (4, 0), (3, 4), (4, 1)])
def test_launch_multi_matches_oracle(cuda, oracle_mod, family, params, ndev, halo):
    """pk_launch_multi over 'devices' that all map to GPU 0 (separate buffers,
    peer copies become device copies): shares, ghost-zone exchanges and the
    gather give the oracle's result on devices[0].  halo = 0: the stencils'
    exchange fused into the sweep (edge blocks store into the neighbours'
    buffers, device counters order the devices); halo > 0: ghost zones of
    that width refreshed by peer copies."""
    from paper_1801_04348_b200 import programs, run_program

    kind = programs.original(family)
    shapes = programs.array_shapes(kind, params)
    rng = np.random.default_rng(ndev * 7 + halo)
    init = {}
    for k, s in shapes.items():
        if family == "jacobi" or family == "jacobi2d":
            init[k] = rng.integers(-(2**31), 2**31 - 1, size=s).astype(np.int32) if halo == 1 or ndev == 4 else \
                rng.integers(-1000, 1000, size=s).astype(np.int32)
        else:
            init[k] = rng.integers(-40, 40, size=s).astype(np.int32)
    want = oracle_mod.run(family, params, init)
    got = run_program(programs.source(family), params, init, devices=[0] * ndev, halo=halo)
    for name in programs.FAMILIES[family].written:
        assert np.array_equal(np.asarray(got[name]).reshape(-1), np.asarray(want[name]).reshape(-1)), name


@pytest.mark.parametrize("family,params", [
    ("reverse", {"N": 0, "s": 2, "B": 32}), ("reverse", {"N": 5, "s": 2, "B": 32}),
    ("matmul", {"n": 0, "B0": 4, "ub1": 2, "s": 2}), ("matmul", {"n": 3, "B0": 4, "ub1": 2, "s": 2}),
    ("matvec", {"N": 0, "s": 1, "B": 32}), ("transpose", {"N": 3, "s": 2, "B0": 4, "B1": 4}),
    ("addition", {"N": 0, "B0": 2, "B1": 2}),
    ("jacobi", {"T": 3, "N": 2, "s": 1, "B": 4}), ("jacobi", {"T": 0, "N": 50, "s": 1, "B": 4}),
    ("jacobi", {"T": 5, "N": 1001, "s": 2, "B": 32}),
    ("jacobi2d", {"T": 2, "N": 2, "s": 1, "B0": 2, "B1": 2}), ("jacobi2d", {"T": 3, "N": 67, "s": 2, "B0": 4, "B1": 8}),
])
def test_run_host_edge_sizes_match_oracle(cuda, oracle_mod, family, params):
    """The host-buffer entry point on empty arrays, extents below one block,
    T = 0, stencils without interior and odd stencil sizes: the host
    buffers end as the oracle leaves them."""
    from paper_1801_04348_b200 import _lib, binding, cases, programs

    kind = programs.original(family)
    shapes = programs.array_shapes(kind, params)
    rng = np.random.default_rng(21)
    init = {k: rng.integers(-1000, 1000, size=s).astype(np.int32) for k, s in shapes.items()}
    want = oracle_mod.run(family, params, init)
    host = {k: np.ascontiguousarray(v.copy()) for k, v in init.items()}
    sel = cases.select(kind, params, "nominal")
    L = binding.make_launch(kind, params, sel.applied)
    _lib.run_host(L, [host[a.name].ctypes.data for a in programs.FAMILIES[family].arrays], 0)
    for name in shapes:
        assert np.array_equal(host[name].reshape(-1), np.asarray(want[name]).reshape(-1)), name


@pytest.mark.parametrize("family,params", [
    ("reverse", {"N": 0, "s": 2, "B": 32}), ("reverse", {"N": 200, "s": 2, "B": 32}),
    ("matmul", {"n": 0, "B0": 4, "ub1": 2, "s": 2}), ("matmul", {"n": 9, "B0": 4, "ub1": 2, "s": 2}),
    ("matvec", {"N": 5, "s": 1, "B": 2}), ("transpose", {"N": 6, "s": 1, "B0": 2, "B1": 2}),
    ("jacobi", {"T": 3, "N": 2, "s": 1, "B": 4}), ("jacobi", {"T": 4, "N": 14, "s": 1, "B": 4}),
    ("jacobi", {"T": 0, "N": 50, "s": 1, "B": 4}),
    ("jacobi2d", {"T": 2, "N": 2, "s": 1, "B0": 2, "B1": 2}), ("jacobi2d", {"T": 3, "N": 8, "s": 1, "B0": 2, "B1": 2}),
])
@pytest.mark.parametrize("ndev", [3, 4])
def test_launch_multi_fewer_units_than_devices(cuda, oracle_mod, family, params, ndev):
    """More devices than units (some devices get empty shares), empty arrays,
    T = 0, stencils without interior: the oracle's result on devices[0]."""
    from paper_1801_04348_b200 import programs, run_program

    kind = programs.original(family)
    shapes = programs.array_shapes(kind, params)
    rng = np.random.default_rng(ndev)
    init = {k: rng.integers(-1000, 1000, size=s).astype(np.int32) for k, s in shapes.items()}
    want = oracle_mod.run(family, params, init)
    got = run_program(programs.source(family), params, init, devices=[0] * ndev)
    for name in shapes:
        assert np.array_equal(np.asarray(got[name]).reshape(-1), np.asarray(want[name]).reshape(-1)), name


@pytest.mark.parametrize("family,params", [
    ("jacobi", {"T": 501, "N": (1 << 20) + 2, "s": 4, "B": 256}),
    ("jacobi2d", {"T": 500, "N": 1026, "s": 4, "B0": 8, "B1": 32}),
])
@pytest.mark.parametrize("ndev", [2, 4])
def test_fused_peer_sweeps_under_real_concurrency(cuda, family, params, ndev):
    """pk_launch_multi's fused sweep with every "device" a separate stream on
    the one GPU: the devices' kernels run truly concurrently (unlike separate
    processes, which time-slice), so the edge blocks' waits and signals race
    the neighbours' stores for hundreds of steps.  Bit-identical to one
    pk_launch of the whole program."""
    torch = cuda
    from paper_1801_04348_b200 import programs, run_program

    N = params["N"]
    n = 2 * N if family == "jacobi" else 2 * N * N
    g = torch.Generator(device="cuda").manual_seed(ndev)
    a = torch.randint(-(1 << 20), 1 << 20, (n,), dtype=torch.int32, device="cuda", generator=g)
    if family == "jacobi2d":
        a = a.view(2 * N, N)
    want = run_program(programs.source(family), params, {"a": a})["a"]
    for _ in range(3):
        got = run_program(programs.source(family), params, {"a": a}, devices=[0] * ndev)["a"]
        assert torch.equal(got.reshape(-1), want.reshape(-1))
