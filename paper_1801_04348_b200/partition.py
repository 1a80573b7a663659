"""Partitioner: one process per GPU, each owning a slice of the program's units.

SURVEY 8(e).  Every rank holds full-size arrays with the program's own
global indexing (memory is not the constraint: the largest BASELINE
instance is 8 GiB against 180 GB of HBM per GPU) and runs the selected
leaf on its unit range through ``pk_launch``'s ``lo``/``hi`` fields:

* reverse    -- input elements p (output range mirrored); no exchange
* transpose  -- rows of c; every rank reads a's column slab in place
* matvec     -- rows of a / y (x replicated)
* matmul     -- rows of a / c (b replicated)
* addition   -- rows
* jacobi     -- interior positions 1..P; ghost zones of width h refreshed
               every h steps with NCCL send/recv, the steps in between
               computed redundantly on the shrinking overlap
* jacobi2d   -- interior rows 1..I; ghost rows likewise

Only the stencils exchange data (a real dependence); the others shard with
no data-path collective.  Ranges are aligned to the leaf's block tile so
each rank launches whole tiles.

Communication goes through an ``Exchanger``: ``TorchExchanger`` uses
torch.distributed point-to-point ops (NCCL over NVLink on GPUs, gloo on
CPU for tests); ``LocalExchanger`` pairs in-process ranks (single-GPU
simulation of a multi-rank run).
"""

from __future__ import annotations

from dataclasses import dataclass

from . import programs

ROW_FAMILIES = ("transpose", "matvec", "matmul", "addition")
SHARDED_FAMILIES = ("reverse",) + ROW_FAMILIES  # run_rows


from .programs import c_div as _c_div  # noqa: E402  (interp.py:43-46)


def units(family: str, P: dict) -> tuple[int, int, int]:
    """(first unit, end unit, alignment) of the work the program covers."""
    if family == "reverse":
        tile = P["s"] * P["B"]
        return 0, max(0, _c_div(P["N"], tile)) * tile, 4 * tile
    if family == "transpose":
        return 0, max(0, _c_div(P["N"], P["B0"])) * P["B0"], max(P["B0"], 4)
    if family == "matvec":
        tile = P["s"] * P["B"]
        return 0, max(0, _c_div(P["N"], tile)) * tile, tile
    if family == "matmul":
        return 0, max(0, _c_div(P["n"], P["B0"])) * P["B0"], max(P["B0"], 4)
    if family == "addition":
        return 0, max(0, _c_div(P["N"], P["B0"])) * P["B0"], P["B0"]
    if family == "jacobi":
        tile = P["s"] * P["B"]
        return 1, 1 + max(0, _c_div(P["N"] - 2, tile)) * tile, tile
    if family == "jacobi2d":
        return 1, 1 + max(0, _c_div(P["N"] - 2, P["B0"])) * P["B0"], P["B0"]
    raise KeyError(family)


def split(family: str, P: dict, rank: int, world: int) -> tuple[int, int]:
    """This rank's contiguous unit range; ranges tile [first, end) exactly,
    boundaries on multiples of the alignment where the extent allows."""
    first, end, align = units(family, P)
    total = end - first
    if total <= 0 or world <= 1:
        return first, end
    blocks = total // align if align > 0 else total
    if blocks >= world and align > 0:
        lo_b = blocks * rank // world
        hi_b = blocks * (rank + 1) // world
        lo = first + lo_b * align
        hi = first + hi_b * align if rank < world - 1 else end
        return lo, hi
    lo = first + total * rank // world
    hi = first + total * (rank + 1) // world
    return lo, hi


# --------------------------------------------------------------- exchange ---

class Exchanger:
    """Point-to-point exchange of equally shaped tensor slices."""

    rank: int
    world: int

    def exchange(self, ops: list[tuple[str, object, int]]) -> None:
        """ops: ('send' | 'recv', tensor, peer).  Blocks until complete."""
        raise NotImplementedError


class TorchExchanger(Exchanger):
    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def exchange(self, ops):
        d = self.dist
        # gloo moves host memory only: CUDA slices are staged through host copies
        staged = d.get_backend(self.group) == "gloo"
        p2p, back = [], []
        for kind, t, peer in ops:
            buf = t
            if staged and t.is_cuda:
                buf = t.cpu() if kind == "send" else t.new_empty(t.shape, device="cpu")
                if kind == "recv":
                    back.append((t, buf))
            fn = d.isend if kind == "send" else d.irecv
            p2p.append(d.P2POp(fn, buf, peer, group=self.group))
        if p2p:
            for req in d.batch_isend_irecv(p2p):
                req.wait()
        for t, buf in back:
            t.copy_(buf)


class LocalExchanger(Exchanger):
    """In-process ranks sharing one mailbox (single-device simulation)."""

    def __init__(self, rank: int, world: int, mailbox: dict):
        self.rank, self.world, self.box = rank, world, mailbox

    def exchange(self, ops):
        for kind, t, peer in ops:
            if kind == "send":
                seq = self.box.get("seq", 0)
                self.box["seq"] = seq + 1
                self.box[(self.rank, peer, seq)] = t.clone()
        self._pending = [(t, peer) for kind, t, peer in ops if kind == "recv"]

    def complete(self):
        for t, peer in self._pending:
            keys = sorted(k for k in self.box if k != "seq" and k[0] == peer and k[1] == self.rank)
            t.copy_(self.box.pop(keys[0]))
        self._pending = []


# ---------------------------------------------------------------- stencils --

@dataclass
class HaloPlan:
    lo: int
    hi: int
    first: int
    end: int
    width: int  # ghost width h: steps per exchange


def halo_plan(family: str, P: dict, rank: int, world: int, width: int | None = None) -> HaloPlan:
    lo, hi = split(family, P, rank, world)
    first, end, _ = units(family, P)
    sizes = [split(family, P, r, world) for r in range(world)]
    min_size = min(h - l for l, h in sizes) if sizes else 0
    h = width if width is not None else 16
    h = max(1, min(h, max(1, min_size), max(1, P["T"])))
    return HaloPlan(lo, hi, first, end, h)


def halves(family: str, a, N: int):
    """(half0, half1) views of the flat double buffer."""
    if family == "jacobi":
        return a[:N], a[N:2 * N]
    return a[: N * N], a[N * N: 2 * N * N]


def src_dst(family: str, t: int, h0, h1):
    """Which half step t reads and writes.  1-D: t even writes a[p+1] from
    the upper half (jacobi.mfk:19-23); 2-D: t even writes a[N+i][j] from the
    lower half."""
    even = t % 2 == 0
    if family == "jacobi":
        return (h1, h0) if even else (h0, h1)
    return (h0, h1) if even else (h1, h0)


def run_stencil(family: str, P: dict, a, ex: Exchanger, sweep, *, width: int | None = None,
                plan: HaloPlan | None = None):
    """Run T steps of a Jacobi program on this rank's slab.

    ``a``: this rank's full-size flat buffer (global indexing).  ``sweep(src,
    dst, lo, hi)`` runs one step over units [lo, hi) (pk_jacobi_sweep on the
    GPU).  Every ``width`` steps the ghost units of the source half are
    refreshed from the neighbours; the steps in between also recompute the
    overlap, shrinking it by one unit per step.
    """
    N, T = P["N"], P["T"]
    plan = plan or halo_plan(family, P, ex.rank, ex.world, width)
    h0, h1 = halves(family, a, N)
    row = 1 if family == "jacobi" else N  # elements per unit
    t = 0
    while t < T:
        hb = min(plan.width, T - t)
        src, _ = src_dst(family, t, h0, h1)
        ops = []
        if ex.rank > 0:
            ops.append(("send", src[plan.lo * row:(plan.lo + hb) * row], ex.rank - 1))
            ops.append(("recv", src[(plan.lo - hb) * row:plan.lo * row], ex.rank - 1))
        if ex.rank < ex.world - 1:
            ops.append(("send", src[(plan.hi - hb) * row:plan.hi * row], ex.rank + 1))
            ops.append(("recv", src[plan.hi * row:(plan.hi + hb) * row], ex.rank + 1))
        if ex.world > 1:
            ex.exchange(ops)
            if hasattr(ex, "complete"):
                yield "exchanged"
                ex.complete()
        for k in range(hb):
            ext = hb - 1 - k
            lo_k = max(plan.first, plan.lo - ext)
            hi_k = min(plan.end, plan.hi + ext)
            s, d = src_dst(family, t + k, h0, h1)
            sweep(s, d, lo_k, hi_k)
        t += hb
    return


def drive(gen):
    """Run a run_stencil generator to completion (single-rank / torch path)."""
    for _ in gen:
        pass


def drive_local(gens):
    """Lock-step several in-process ranks (LocalExchanger) to completion."""
    alive = list(gens)
    while alive:
        nxt = []
        for g in alive:
            try:
                next(g)
                nxt.append(g)
            except StopIteration:
                pass
        alive = nxt


class PeerStencil:
    """T steps of a Jacobi program with the halo exchange fused into the sweep
    (pk_jacobi_sweep_peer): one process per GPU, every rank holding the whole
    double buffer ``a`` (global indexing) and owning ``split(...)``'s units.
    The blocks that compute a rank's first / last unit also store it into the
    neighbour's buffer through a CUDA IPC mapping (NVLink peer stores between
    B200s) and order themselves against the neighbour with counters in device
    memory -- no NCCL call, no separate exchange step, ghost width 1.

    ``group``: any torch.distributed group (gloo or NCCL) used once to trade
    IPC handles; ``launch``: the pk_launch_t of the selected leaf.
    """

    def __init__(self, family: str, P: dict, a, launch, group=None):
        import torch
        import torch.distributed as dist

        from . import _lib

        if family not in ("jacobi", "jacobi2d"):
            raise ValueError("PeerStencil: %s is not a Jacobi stencil" % family)
        self._lib, self._torch, self._dist = _lib, torch, dist
        self.family, self.P, self.a, self.L, self.group = family, P, a, launch, group
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        self.lo, self.hi = split(family, P, self.rank, self.world)
        # every rank's edge blocks signal its neighbours each step: an empty
        # slab would leave them waiting
        if any(h <= l for l, h in (split(family, P, r, self.world) for r in range(self.world))):
            raise ValueError("PeerStencil: %d ranks for %s leave a rank without units" % (self.world, family))
        # [from_left, from_right, error] in this rank's memory
        self.ctr = torch.zeros(3, dtype=torch.int32, device=a.device)
        mine = (_lib.ipc_export(a.data_ptr()), _lib.ipc_export(self.ctr.data_ptr()))
        every = [None] * self.world
        dist.all_gather_object(every, mine, group=group)
        self._opened = []
        peer = _lib.PkPeer()
        base = self.ctr.data_ptr()
        peer.wait_left, peer.wait_right, peer.error = base, base + 4, base + 8
        if self.rank > 0:
            (ha, oa), (hc, oc) = every[self.rank - 1]
            peer.left_base = self._open(ha, oa)
            peer.signal_left = self._open(hc, oc) + 4  # the left neighbour's from_right
        if self.rank < self.world - 1:
            (ha, oa), (hc, oc) = every[self.rank + 1]
            peer.right_base = self._open(ha, oa)
            peer.signal_right = self._open(hc, oc)  # the right neighbour's from_left
        self.peer = peer

    def _open(self, handle: bytes, offset: int) -> int:
        ptr = self._lib.ipc_open(handle, offset)
        self._opened.append((ptr, offset))
        return ptr

    def run(self, T: int, stream=None) -> None:
        """Steps 0..T-1 (counters zeroed and every rank synchronised first)."""
        torch, dist = self._torch, self._dist
        self.ctr.zero_()
        torch.cuda.synchronize(self.a.device)
        dist.barrier(group=self.group)
        st = stream if stream is not None else torch.cuda.current_stream(self.a.device).cuda_stream
        for t in range(T):
            self._lib.jacobi_sweep_peer(self.L, self.a.data_ptr(), t, self.lo, self.hi, self.peer, st)

    def finish(self) -> None:
        """Wait for every rank (neighbours may still be storing into our buffer)
        and raise if a wait gave up."""
        torch, dist = self._torch, self._dist
        torch.cuda.synchronize(self.a.device)
        # every rank learns whether any wait gave up, so all of them raise together
        # (one rank raising alone would leave the others in the next collective)
        err = torch.tensor([int(self.ctr[2].item())], dtype=torch.int64)
        if dist.get_backend(self.group) == "nccl":
            err = err.to(self.a.device)
        dist.all_reduce(err, op=dist.ReduceOp.MAX, group=self.group)
        if int(err.item()) != 0:
            raise RuntimeError("PeerStencil: a neighbour never signalled (wait timed out)")

    def close(self) -> None:
        self.finish()
        for ptr, off in self._opened:
            self._lib.ipc_close(ptr, off)
        self._opened = []


# ------------------------------------------------------- row-sharded runs --

# operands every rank needs whole (matmul's b, mat-vec's x, the
# transpose source); everything else is cut by the unit range
REPLICATED = {"transpose": ("a",), "matvec": ("x",), "matmul": ("b",)}


def share_range(family: str, P: dict, name: str, lo: int, hi: int) -> tuple[int, int]:
    """(offset, count) in elements of the flat array ``name`` that units
    [lo, hi) read or write -- the rule pk_run_host uses (array_range in
    csrc/pk_abi.cu) to move only a rank's share."""
    N = P["n"] if family == "matmul" else P["N"]
    N = max(0, N)
    total = {n: _numel(d) for n, d in programs.array_shapes(programs.original(family), P).items()}[name]
    if name in REPLICATED.get(family, ()):
        a, b = 0, total
    elif family == "reverse":
        a, b = (lo, hi) if name == "a" else (N - hi, N - lo)
    elif family == "matvec" and name == "y":
        a, b = lo, hi
    elif family in ("transpose", "matvec", "matmul", "addition"):
        a, b = lo * N, hi * N
    else:
        raise KeyError("%s is not a row-sharded family" % family)
    a, b = max(0, a), min(total, b)
    return a, max(0, b - a)


def _numel(dims) -> int:
    n = 1
    for d in dims:
        n *= max(0, d)
    return n


def run_rows(family: str, P: dict, arrays: dict, launch, *, group=None, root: int = 0) -> None:
    """Run a row-sharded family over the ranks of ``group``, in place.

    ``arrays``: name -> this rank's full-size flat tensor (the inputs are
    read on ``root``).  ``launch(lo, hi)`` runs the selected leaf on units
    [lo, hi) over those tensors (``pk_launch`` with lo/hi on the GPU).
    Data movement is done once, outside the compute: the replicated operands
    are broadcast from root, every other rank receives its share of the
    sharded ones point-to-point, and the written shares (plus the uncovered
    tail the program leaves untouched) are broadcast from their owners, so
    every rank ends with the whole result.  The compute itself has no
    collective.
    """
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    fam = programs.FAMILIES[family]
    names = [a.name for a in fam.arrays]
    ranges = [split(family, P, r, world) for r in range(world)]
    if world > 1:
        for name in REPLICATED.get(family, ()):
            dist.broadcast(arrays[name], src=root, group=group)
        ops = []
        for name in names:
            if name in REPLICATED.get(family, ()):
                continue
            for r in range(world):
                off, cnt = share_range(family, P, name, *ranges[r])
                if r == root or cnt == 0:
                    continue
                view = arrays[name][off:off + cnt]
                if rank == root:
                    ops.append(dist.P2POp(dist.isend, view, r, group=group))
                elif rank == r:
                    ops.append(dist.P2POp(dist.irecv, view, root, group=group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
    lo, hi = ranges[rank]
    if hi > lo:
        launch(lo, hi)
    if world > 1:
        first, end, _ = units(family, P)
        for name in fam.written:
            for r in range(world):
                off, cnt = share_range(family, P, name, *ranges[r])
                if cnt:
                    dist.broadcast(arrays[name][off:off + cnt], src=r, group=group)
            # elements no rank covers keep their input values: root's
            off, cnt = share_range(family, P, name, first, end)
            total = arrays[name].numel()
            for a, b in ((0, off), (off + cnt, total)):
                if b > a:
                    dist.broadcast(arrays[name][a:b], src=root, group=group)


def pk_launcher(family: str, P: dict, arrays: dict, *, machine=None, dtype=None, stream=None):
    """``launch(lo, hi)`` for run_rows on the GPU: the case selected at the
    live device, bound to its kernel, launched over units [lo, hi) of the
    caller's CUDA tensors (pk_launch with lo/hi)."""
    import torch

    from . import _lib, binding, cases

    from . import machine as machine_mod

    kind = programs.original(family)
    names = [a.name for a in programs.FAMILIES[family].arrays]
    if dtype is None:
        dtype = {torch.float32: _lib.DTYPE_F32, torch.float64: _lib.DTYPE_F64,
                 torch.int64: _lib.DTYPE_I64}.get(arrays[names[0]].dtype, _lib.DTYPE_I32)
    if machine is None:  # this rank's own device (not device 0): selection on the GPU that runs the leaf
        dev = arrays[names[0]].device
        elem = 8 if dtype in (_lib.DTYPE_F64, _lib.DTYPE_I64) else 4
        machine = machine_mod.live(dev.index if dev.type == "cuda" else torch.cuda.current_device(),
                                   elem_bytes=elem)
    sel = cases.select(kind, P, machine)

    def launch(lo, hi):
        L = binding.make_launch(kind, P, sel.applied, dtype, lo=lo, hi=hi)
        st = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        _lib.launch(L, [arrays[n].data_ptr() for n in names], st)
    return launch


def unit_range_launch(family: str, P: dict, rank: int, world: int) -> tuple[int, int]:
    """lo/hi for pk_launch on rank's share (row / element families)."""
    lo, hi = split(family, P, rank, world)
    if hi <= lo:
        return 0, -1  # empty share: caller skips the launch
    return lo, hi


__all__ = [
    "units", "split", "halo_plan", "run_stencil", "drive", "drive_local", "TorchExchanger",
    "LocalExchanger", "Exchanger", "unit_range_launch", "ROW_FAMILIES", "programs",
    "REPLICATED", "share_range", "run_rows", "pk_launcher", "SHARDED_FAMILIES", "PeerStencil",
]
