"""Leaf-to-kernel binding: a selected case becomes one pk_launch_t.

A case's ``applied`` strategy tuple (engine.py:61-72, 128-151) says which
program variant the leaf runs.  Only the source-level strategies change the
kernel:

* ``granularity`` (strategies.py:302-422) removes the s loop: one element
  per thread, a block tile of B (not s*B) -> PK_FLAG_GRANULARITY.  For the
  addition program it merges the twin stores instead -> PK_FLAG_MERGED when
  the merged TEXT is what the caller runs.
* ``caching-off`` (strategies.py:430-440) drops ``cache(...)``: the kernel
  reads global memory directly -> PK_VARIANT_DIRECT; otherwise tiles are
  staged in shared memory -> PK_VARIANT_STAGED.
* ``cse-*`` / ``regpressure-*`` are IR rewrites of the register estimate;
  nvcc performs the equivalent, so they bind to the same kernel.

The covered index sets always come from the ORIGINAL program's parameters
(the kernels evaluate its bindings with C division), so every leaf writes
exactly the elements the reference interpreter writes.
"""

from __future__ import annotations

from . import _lib
from .programs import FAMILIES, ProgramKind


def make_launch(
    kind: ProgramKind,
    params: dict,
    applied: tuple[str, ...],
    dtype: int = _lib.DTYPE_I32,
    *,
    generic: bool = False,
    lo: int = 0,
    hi: int = 0,
    extra_flags: int = 0,
) -> _lib.PkLaunch:
    fam = FAMILIES[kind.family]
    P = params
    L = _lib.PkLaunch()
    L.family = _lib.FAMILY_IDS[kind.family]
    L.variant = _lib.VARIANT_DIRECT if "caching-off" in applied else _lib.VARIANT_STAGED
    L.dtype = dtype
    flags = extra_flags
    if kind.family == "addition":
        if "granularity" in kind.applied:
            flags |= _lib.FLAG_MERGED
    elif "granularity" in applied:
        flags |= _lib.FLAG_GRANULARITY
    if generic:
        flags |= _lib.FLAG_GENERIC
    L.flags = flags
    L.N = int(P["n"] if kind.family == "matmul" else P["N"])
    L.T = int(P.get("T", 0))
    L.s = int(P.get("s", 1))
    L.B = int(P.get("B", 0))
    L.B0 = int(P.get("B0", 0))
    L.B1 = int(P.get("B1", 0))
    L.ub1 = int(P.get("ub1", 0))
    L.lo = int(lo)
    L.hi = int(hi)
    L.tblock = 0
    assert set(fam.params) <= set(P), (fam.params, P)
    return L


def describe(L: _lib.PkLaunch) -> dict:
    d = L.as_dict()
    d["family"] = {v: k for k, v in _lib.FAMILY_IDS.items()}[L.family]
    d["variant"] = "direct" if L.variant == _lib.VARIANT_DIRECT else "staged"
    d["dtype"] = _lib.DTYPE_NAMES.get(L.dtype, str(L.dtype))
    return d
