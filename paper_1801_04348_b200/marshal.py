"""Host values <-> typed device words, with the reference interpreter's value
semantics.

The reference stores Python objects in Python lists (interp.py:76-81,
183-206): ``_put`` moves the fetched object unchanged, ints never overflow,
floats are binary64.  The kernels see flat buffers of one element type
(``PK_DTYPE_*``, include/pk.h).  This module picks that type per call so the
result equals the reference's, and refuses (loudly) where it cannot:

* **reverse, transpose** move values without computing.  int lists within
  int32 travel as 4-byte words; any other list content (binary64 floats,
  ints beyond int32, bools, mixed types, any object) travels as 8-byte
  *object indices* into a pool of the caller's objects, so every value comes
  back as the very object the reference would have moved (int 0 where an
  unsupplied array was never written).  numpy / torch arrays move as words
  of their own size (4 or 8 bytes; narrower types are widened losslessly)
  and come back in the caller's dtype.
* **addition, matvec, matmul** compute ``c + a*b``-style sums.  Python floats
  and float64 arrays run in binary64 with the interpreter's rounding
  sequence (PK_DTYPE_F64: bit-identical); float32 arrays run the float32
  path the BASELINE configs name (FFMA matmul, double-float mat-vec).  Ints
  run in int32 when a bound on every result proves int32 holds it (two's
  complement sums are exact modulo 2^32, so the final value is exact), in
  int64 when the bound fits int64, and raise ``OverflowError`` beyond that.
* **jacobi, jacobi2d**: ints within int32 run the int32 register sweeps
  (exact 64-bit sums where 32 bits could wrap), wider ints int64 sweeps;
  Python floats / float data run binary64 sweeps whose "/" is the
  reference's c_div on floats (interp.py:43-46: CPython's float floor
  division of the absolute values, with the sign) -- bit-identical.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib

WORD_FAMILIES = ("reverse", "transpose")
ARITH_FAMILIES = ("addition", "matvec", "matmul")
INT_FAMILIES = ("jacobi", "jacobi2d")

I32_MIN, I32_MAX = -(2**31), 2**31 - 1
I64_MIN, I64_MAX = -(2**63), 2**63 - 1

NP_OF_DTYPE = {
    _lib.DTYPE_I32: np.dtype(np.int32),
    _lib.DTYPE_F32: np.dtype(np.float32),
    _lib.DTYPE_I64: np.dtype(np.int64),
    _lib.DTYPE_F64: np.dtype(np.float64),
}


def kind_of(value) -> str:
    if isinstance(value, np.ndarray):
        return "numpy"
    if type(value).__module__.startswith("torch"):
        return "torch"
    return "list"


def _flatten_list(value) -> list:
    if value and isinstance(value[0], (list, tuple)):
        return [v for row in value for v in row]
    return list(value)


@dataclass
class Source:
    """One array the caller supplied."""

    name: str
    value: object
    kind: str  # list | numpy | torch
    vkind: str  # int | float | mixed | object | f32 | f64 | i (numpy/torch ints)
    lo: int = 0  # value range (ints)
    hi: int = 0
    flat: object = None  # list: the flat Python values; numpy: flat ndarray
    size: int = 0
    np_dtype: object = None  # numpy / torch: the caller's element type (numpy dtype)


def _torch_np_dtype(t):
    import torch

    table = {torch.float32: np.float32, torch.float64: np.float64, torch.float16: np.float16,
             torch.bfloat16: np.float32, torch.int8: np.int8, torch.int16: np.int16, torch.int32: np.int32,
             torch.int64: np.int64, torch.uint8: np.uint8, torch.bool: np.bool_}
    if t.dtype not in table:
        raise TypeError("arrays of %s are not supported" % t.dtype)
    return np.dtype(table[t.dtype])


def describe(name: str, value) -> Source:
    k = kind_of(value)
    if k == "list":
        flat = _flatten_list(value)
        types = set(map(type, flat))
        if types <= {int}:
            lo, hi = (min(flat), max(flat)) if flat else (0, 0)
            return Source(name, value, k, "int", lo, hi, flat, len(flat))
        if types <= {float}:
            return Source(name, value, k, "float", flat=flat, size=len(flat))
        if types <= {int, float}:
            return Source(name, value, k, "mixed", flat=flat, size=len(flat))
        return Source(name, value, k, "object", flat=flat, size=len(flat))
    if k == "numpy":
        dt = value.dtype
        flat = value.reshape(-1)
        if dt.kind == "f":
            return Source(name, value, k, "f64" if dt.itemsize == 8 else "f32", flat=flat, size=flat.size, np_dtype=dt)
        if dt.kind in "iub":
            lo, hi = (int(flat.min()), int(flat.max())) if flat.size else (0, 0)
            return Source(name, value, k, "i", lo, hi, flat, flat.size, dt)
        if dt.kind == "O":
            return describe(name, value.tolist()) if value.ndim <= 2 else Source(name, value, k, "object",
                                                                                  flat=list(flat), size=flat.size)
        raise TypeError("array %s: numpy dtype %s is not supported" % (name, dt))
    t = value.detach()
    dt = _torch_np_dtype(t)
    if t.is_floating_point():
        return Source(name, value, k, "f64" if dt.itemsize == 8 else "f32", size=t.numel(), np_dtype=dt)
    if t.numel():
        lo, hi = int(t.min()), int(t.max())
    else:
        lo = hi = 0
    return Source(name, value, k, "i", lo, hi, size=t.numel(), np_dtype=dt)


@dataclass
class Plan:
    """How one run_program call maps the caller's values onto device words."""

    family: str
    dtype: int  # PK_DTYPE_*
    objects: bool = False  # permutation of Python objects by index words
    pool: list = field(default_factory=list)  # objects mode: the caller's objects, then int 0
    offsets: dict = field(default_factory=dict)  # objects mode: first pool index of each array
    out_dtype: dict = field(default_factory=dict)  # numpy/torch callers: dtype each array returns in
    default_out: object = None  # ... and the dtype of arrays they did not supply

    @property
    def np_dtype(self) -> np.dtype:
        return NP_OF_DTYPE[self.dtype]

    @property
    def elem_bytes(self) -> int:
        return self.np_dtype.itemsize

    @property
    def zero_index(self) -> int:
        return len(self.pool) - 1


def _abs_max(s: Source) -> int:
    return max(abs(s.lo), abs(s.hi))


def int_bound(family: str, P: dict, srcs: dict) -> int:
    """An upper bound on |value| of every element the program leaves in its
    arrays (inputs included), from the inputs' ranges."""
    m = {n: _abs_max(s) for n, s in srcs.items()}
    get = lambda n: m.get(n, 0)  # noqa: E731 -- unsupplied arrays are zeros
    inputs = max(m.values()) if m else 0
    if family == "addition":
        return max(inputs, get("a") + get("b"))
    if family == "matvec":
        return max(inputs, get("y") + max(0, P["N"]) * get("a") * get("x"))
    if family == "matmul":
        n, B0 = P["n"], P["B0"]
        K = max(0, n // B0) * B0 if B0 > 0 else 0
        return max(inputs, get("c") + K * get("a") * get("b"))
    return inputs


def plan(family: str, P: dict, supplied: dict) -> tuple[Plan, dict]:
    """Choose the element type for a call; returns (plan, {name: Source})."""
    srcs = {n: describe(n, v) for n, v in supplied.items()}
    vkinds = {s.vkind for s in srcs.values()}
    if family in WORD_FAMILIES:
        if any(s.kind == "list" and (s.vkind != "int" or s.lo < I32_MIN or s.hi > I32_MAX)
               for s in srcs.values()) or "object" in vkinds:
            return _objects_plan(family, srcs), srcs
        if not srcs or all(s.kind == "list" for s in srcs.values()):
            return Plan(family, _lib.DTYPE_I32), srcs
        dts = [s.np_dtype if s.np_dtype is not None else np.dtype(np.int32) for s in srcs.values()]
        common = np.result_type(*dts)
        if common.kind == "f":
            dtype = _lib.DTYPE_F64 if common.itemsize == 8 else _lib.DTYPE_F32
        elif common.itemsize == 8:
            dtype = _lib.DTYPE_I64
        else:
            dtype = _lib.DTYPE_I32
        if common.kind == "u" and common.itemsize == 8:
            common = np.dtype(np.uint64)  # moved as 8-byte words, returned as uint64
        return Plan(family, dtype, out_dtype={n: common for n in srcs}, default_out=common), srcs
    if "object" in vkinds:
        bad = next(s for s in srcs.values() if s.vkind == "object")
        raise TypeError("array %s holds values that are neither int nor float; %s computes on numbers"
                        % (bad.name, family))
    floats = vkinds & {"float", "mixed", "f32", "f64"}
    if floats:
        # binary64 wherever the reference's Python floats (or float64 data) are
        # involved; float32 data alone run the float32 path -- except for the
        # stencils, whose "/" is c_div on Python floats (binary64 only)
        dtype = _lib.DTYPE_F32 if floats == {"f32"} and family not in INT_FAMILIES else _lib.DTYPE_F64
        out = NP_OF_DTYPE[dtype]
        return Plan(family, dtype, out_dtype={n: out for n in srcs}), srcs
    # integers: the narrowest type that provably holds every result
    for s in srcs.values():
        if s.lo < I64_MIN or s.hi > I64_MAX:
            raise OverflowError("array %s holds values outside int64" % s.name)
    if family in INT_FAMILIES:
        # an average never leaves its inputs' range: int32 data run the int32
        # sweeps (64-bit sums where needed); wider data the int64 sweeps, whose
        # sums of 3 (5) values must fit int64
        wide = any(s.lo < I32_MIN or s.hi > I32_MAX for s in srcs.values())
        if wide and 5 * max(_abs_max(s) for s in srcs.values()) > I64_MAX:
            raise OverflowError("%s: sums of 5 values up to %d leave int64" % (family, max(_abs_max(s) for s in srcs.values())))
        dt = _lib.DTYPE_I64 if wide else _lib.DTYPE_I32
        out = {n: np.result_type(NP_OF_DTYPE[dt], s.np_dtype) if s.np_dtype is not None else NP_OF_DTYPE[dt]
               for n, s in srcs.items()}
        return Plan(family, dt, out_dtype=out), srcs
    bound = int_bound(family, P, srcs)
    if bound <= I32_MAX:
        dtype = _lib.DTYPE_I32
    elif bound <= I64_MAX:
        dtype = _lib.DTYPE_I64
    else:
        raise OverflowError("%s: results may reach %d, beyond int64; the kernels compute in at most 64-bit "
                            "integers" % (family, bound))
    # numpy / torch callers get at least their own integer width back
    out = {n: np.result_type(NP_OF_DTYPE[dtype], s.np_dtype) if s.np_dtype is not None else NP_OF_DTYPE[dtype]
           for n, s in srcs.items()}
    return Plan(family, dtype, out_dtype=out), srcs


def _objects_plan(family: str, srcs: dict) -> Plan:
    pl = Plan(family, _lib.DTYPE_I64, objects=True)
    for n, s in srcs.items():
        flat = s.flat if isinstance(s.flat, list) else (list(s.flat) if s.flat is not None
                                                      else s.value.reshape(-1).tolist())
        s.flat = flat
        pl.offsets[n] = len(pl.pool)
        pl.pool.extend(flat)
    pl.pool.append(0)  # what an unsupplied array holds (interp.py:79-81: [0] * n)
    return pl


def host_words(pl: Plan, src: Source | None, count: int, out: np.ndarray) -> None:
    """Write the first ``count`` elements of an array, as device words, into
    ``out`` (a numpy view of dtype pl.np_dtype, e.g. of pinned memory);
    elements the caller did not supply are zero."""
    import torch

    if src is None:
        if pl.objects:
            out[:count] = pl.zero_index
        else:
            torch.from_numpy(out[:count]).zero_()
        return
    n = min(count, src.size)
    if pl.objects:
        base = pl.offsets[src.name]
        out[:n] = np.arange(base, base + n, dtype=np.int64)
        out[n:count] = pl.zero_index
        return
    if src.kind == "list":
        arr = np.asarray(src.flat[:n], dtype=np.float64 if pl.np_dtype.kind == "f" else np.int64)
        out[:n] = arr.astype(pl.np_dtype, copy=False)
    elif src.kind == "numpy":
        a = src.flat[:n]
        if a.dtype != pl.np_dtype:
            a = _retype(a, pl.np_dtype)
        torch.from_numpy(out[:n]).copy_(torch.from_numpy(np.ascontiguousarray(a)))  # multi-threaded copy
    else:
        t = src.value.detach().reshape(-1)[:n]
        dst = torch.from_numpy(out[:n])
        if t.dtype == _torch_dtype(pl.np_dtype):
            dst.copy_(t)
        else:
            dst.copy_(torch.from_numpy(_retype(t.cpu().numpy(), pl.np_dtype)))
    if n < count:
        torch.from_numpy(out[n:count]).zero_()


def _retype(a: np.ndarray, dt: np.dtype) -> np.ndarray:
    """Values of ``a`` as ``dt`` words: a bit view where the sizes agree and
    the plan moves words (permutations), a value conversion otherwise."""
    if a.dtype.itemsize == dt.itemsize and (a.dtype.kind == dt.kind or a.dtype.kind in "iu" and dt.kind in "iu"):
        return a.view(dt)
    return a.astype(dt)


def _torch_dtype(dt: np.dtype):
    import torch

    return {np.dtype(np.int32): torch.int32, np.dtype(np.int64): torch.int64, np.dtype(np.float32): torch.float32,
            np.dtype(np.float64): torch.float64}[np.dtype(dt)]


def _torch_out_dtype(dt: np.dtype):
    import torch

    table = {np.float32: torch.float32, np.float64: torch.float64, np.float16: torch.float16, np.int8: torch.int8,
             np.int16: torch.int16, np.int32: torch.int32, np.int64: torch.int64, np.uint8: torch.uint8,
             np.bool_: torch.bool}
    return table.get(np.dtype(dt).type, _torch_dtype(dt) if np.dtype(dt).itemsize in (4, 8) else torch.float32)


def torch_dtype(pl: Plan):
    return _torch_dtype(pl.np_dtype)


def device_words(pl: Plan, src: Source, count: int, device):
    """A fresh device tensor of ``count`` elements of the plan's type holding
    the caller's array (torch inputs: converted on their own device)."""
    import torch

    td = torch_dtype(pl)
    if src.kind == "torch" and not pl.objects:
        t = src.value.detach().reshape(-1)
        n = min(count, t.numel())
        out = torch.zeros(max(count, 1), dtype=td, device=device)
        part = t[:n].to(device)
        if part.dtype != td:
            if pl.family in WORD_FAMILIES and part.element_size() == out.element_size():
                part = part.view(td)
            else:
                part = part.to(td)
        out[:n].copy_(part)
        return out
    host = np.empty(max(count, 1), dtype=pl.np_dtype)
    host_words(pl, src, count, host)
    return torch.from_numpy(host).to(device)


def finish(pl: Plan, src: Source | None, words, shape, like_kind: str, like=None, owned: bool = False):
    """The caller-facing array for one program array.

    ``words``: flat numpy array (host) or torch tensor (device) holding the
    declared elements after the run.  Elements the caller supplied beyond the
    declared extent are returned unchanged; the container is the caller's
    (list / numpy / torch on the caller's device), numpy and torch arrays in
    ``pl.out_dtype`` (the caller's dtype for the permutations).  ``owned``:
    ``words`` is a fresh host array this call may hand out without a copy.
    """
    count = 1
    for d in shape:
        count *= d
    if src is not None and src.size < count:  # shorter than declared, long enough for every access
        count, shape = src.size, (src.size,)
    extra = src.size - count if src is not None and src.size > count else 0
    if pl.objects:
        idx = words if isinstance(words, np.ndarray) else words.cpu().numpy()
        vals = [pl.pool[i] for i in idx[:count].tolist()]
        if extra:
            vals += src.flat[count:]
            return _as_kind(vals, (len(vals),), like_kind, object)
        return _as_kind(vals, shape, like_kind, object)
    out_dt = pl.out_dtype.get(src.name) if src is not None else pl.default_out
    if out_dt is None:
        out_dt = pl.np_dtype
    if like_kind == "torch":
        import torch

        t = words if not isinstance(words, np.ndarray) else torch.from_numpy(words)
        t = t[:count]
        if extra:
            rest = src.value.detach().reshape(-1)[count:].to(t.device)
            t = torch.cat([t, rest.to(t.dtype) if rest.dtype != t.dtype else rest])
        if out_dt != pl.np_dtype:
            ot = _torch_out_dtype(out_dt)
            t = t.view(ot) if out_dt.itemsize == pl.np_dtype.itemsize and out_dt.kind == pl.np_dtype.kind else t.to(ot)
        dev = like.device if like is not None else t.device
        t = t.to(dev)
        return t.reshape(shape) if not extra else t
    host = words if isinstance(words, np.ndarray) else words.cpu().numpy()
    host = host[:count]
    if out_dt != pl.np_dtype:  # the caller's dtype: same-size words as a view, narrower ones converted back
        host = host.view(out_dt) if out_dt.itemsize == pl.np_dtype.itemsize else host.astype(out_dt)
    if extra:
        tail = src.flat[count:] if src.kind == "list" else src.value.reshape(-1)[count:]
        if like_kind == "list":
            return host.tolist() + list(tail)
        return np.concatenate([host, np.asarray(tail).astype(host.dtype)])
    if like_kind == "numpy":
        return host.reshape(shape) if owned else host.reshape(shape).copy()
    return host.reshape(shape).tolist()


def copy_input(pl: Plan, src: Source | None, shape, like_kind: str, like=None):
    """The caller-facing value of an array the program never writes: a copy
    of what the caller supplied (interp.py:183-186 deep-copies inputs), in
    the dtype finish() would return it in, without a device round trip.
    Lists come back as lists of the very same objects (an int stays an int
    even when the run computes in binary64)."""
    import torch

    count = 1
    for d in shape:
        count *= d
    if src is None:
        if like_kind == "list":
            return [[0] * shape[1] for _ in range(shape[0])] if len(shape) == 2 else [0] * shape[0]
        dt = pl.default_out if pl.default_out is not None else pl.np_dtype
        if like_kind == "numpy":
            return np.zeros(shape, dtype=dt)
        return torch.zeros(shape, dtype=_torch_out_dtype(dt))
    if src.kind == "list":
        v = src.value
        return [list(r) for r in v] if v and isinstance(v[0], (list, tuple)) else list(v)
    out_dt = pl.out_dtype.get(src.name) or pl.np_dtype
    if pl.objects:
        out_dt = None
    if src.kind == "numpy":
        a = src.value
        if out_dt is not None and a.dtype != out_dt:
            return a.astype(out_dt)
        return fresh_copy(a)
    t = src.value.detach()
    if out_dt is not None and t.dtype != _torch_out_dtype(out_dt):
        return t.to(_torch_out_dtype(out_dt))
    return t.clone()


def _par_copy_types():
    import torch

    return {np.dtype(np.float32): torch.float32, np.dtype(np.float64): torch.float64,
            np.dtype(np.int32): torch.int32, np.dtype(np.int64): torch.int64, np.dtype(np.int16): torch.int16,
            np.dtype(np.int8): torch.int8, np.dtype(np.uint8): torch.uint8, np.dtype(np.float16): torch.float16}


class _LazyTypes(dict):
    def get(self, k, default=None):
        if not self:
            self.update(_par_copy_types())
        return super().get(k, default)


_PAR_COPY = _LazyTypes()


def direct_words(pl: Plan, src: Source | None, count: int):
    """The caller's own host array when it already holds the plan's words
    (C-contiguous, the plan's element size, at least ``count`` elements):
    pk_run_host_io can read it in place.  None otherwise."""
    if src is None or pl.objects or src.kind == "list":
        return None
    if src.kind == "numpy":
        a = src.value
    else:
        t = src.value.detach()
        if t.is_cuda or not t.is_contiguous():
            return None
        a = t.numpy()
    if not a.flags.c_contiguous or a.size < count or a.dtype.itemsize != pl.np_dtype.itemsize:
        return None
    if a.dtype != pl.np_dtype and not (pl.family in WORD_FAMILIES and a.dtype.kind in "iuf"):
        return None  # a value conversion is needed (e.g. int64 data for an int64 ... float64 plan)
    return a.reshape(-1)


def finish_copy(arr: np.ndarray, src: Source, shape, like_kind: str, like=None):
    """The caller-facing copy of an unwritten array the library copied into
    ``arr`` (a fresh host array of the caller's element type)."""
    if like_kind == "torch":
        import torch

        return torch.from_numpy(arr.view(src.np_dtype) if arr.dtype != src.np_dtype else arr).reshape(src.value.shape)
    return arr.reshape(src.value.shape)


class HostPool:
    """Recycled host memory for result arrays.

    Writing fresh (never touched) pages costs a page fault per 4 KB: at
    n = 8192 the 768 MB of results a run_program call hands back took ~30 ms
    of faults against ~10 ms of copying into touched memory.  Each result is
    a view of a pooled base buffer; a base is reused only once no array
    refers to it any more (its reference count is back to the pool's own),
    so every array a caller holds stays exclusively theirs.  ``release()``
    returns the memory to the system."""

    def __init__(self, keep_bytes: int = 8 << 30):
        import threading

        self.lock = threading.Lock()
        self.bases: list = []
        self.keep_bytes = keep_bytes

    def take(self, nbytes: int) -> np.ndarray:
        import sys

        import torch

        nbytes = max(int(nbytes), 1)
        with self.lock:
            best = None
            for i in range(len(self.bases)):
                # referenced by the list and getrefcount's argument only: free
                if sys.getrefcount(self.bases[i]) == 2 and nbytes <= self.bases[i].size <= 2 * nbytes:
                    if best is None or self.bases[i].size < self.bases[best].size:
                        best = i
            if best is not None:
                return self.bases[best][:nbytes]
            base = torch.empty(nbytes, dtype=torch.uint8).numpy()
            total = sum(b.size for b in self.bases) + nbytes
            if total <= self.keep_bytes:
                self.bases.append(base)
            return base[:nbytes]

    def release(self) -> None:
        with self.lock:
            self.bases.clear()


host_pool = HostPool()


def fresh_array(count: int, dtype) -> np.ndarray:
    """An uninitialised host array for a result (from the recycled pool)."""
    dt = np.dtype(dtype)
    return host_pool.take(max(count, 1) * dt.itemsize).view(dt)


def fresh_copy(words: np.ndarray) -> np.ndarray:
    """A fresh host array with the contents of ``words`` (e.g. a pinned
    staging buffer), copied by torch's threads (page-faulting fresh memory is
    the slow part of a large copy)."""
    import torch

    td = _PAR_COPY.get(words.dtype)
    if words.size < (1 << 16) or td is None or not words.flags.c_contiguous:
        return words.copy()
    out = torch.empty(words.shape, dtype=td).numpy()
    torch.from_numpy(out).copy_(torch.from_numpy(words))
    return out


def _as_kind(vals: list, shape, like_kind: str, _dt):
    if like_kind == "numpy":
        arr = np.empty(len(vals), dtype=object)
        arr[:] = vals
        return arr.reshape(shape)
    if len(shape) == 2:
        r, c = shape
        return [vals[i * c:(i + 1) * c] for i in range(r)]
    return vals
