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


def _c_div(a: int, b: int) -> int:
    q = abs(a) // abs(b)
    return q if (a >= 0) == (b >= 0) else -q


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
        p2p = []
        for kind, t, peer in ops:
            fn = d.isend if kind == "send" else d.irecv
            p2p.append(d.P2POp(fn, t, peer, group=self.group))
        if p2p:
            for req in d.batch_isend_irecv(p2p):
                req.wait()


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


def unit_range_launch(family: str, P: dict, rank: int, world: int) -> tuple[int, int]:
    """lo/hi for pk_launch on rank's share (row / element families)."""
    lo, hi = split(family, P, rank, world)
    if hi <= lo:
        return 0, -1  # empty share: caller skips the launch
    return lo, hi


__all__ = [
    "units", "split", "halo_plan", "run_stencil", "drive", "drive_local", "TorchExchanger",
    "LocalExchanger", "Exchanger", "unit_range_launch", "ROW_FAMILIES", "programs",
]
