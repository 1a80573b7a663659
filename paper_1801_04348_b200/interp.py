"""Drop-in replacement for ``parakern.interp.run_program`` on sm_100a.

    from paper_1801_04348_b200.interp import run_program
    out = run_program(program, {"N": 1 << 20, "s": 4, "B": 256}, arrays={"a": a})

Same contract as the reference (/root/reference/pkg/src/parakern/interp.py:215-225):

* ``program``: a ``parakern.dsl.Program`` or its ``.mfk`` text;
* ``params``: scalar parameter values; a missing one raises ``KeyError``
  (interp.py:73-75), a zero divisor in a binding ``ZeroDivisionError``;
* ``arrays``: optional initial contents; the caller's buffers are never
  mutated (interp.py:76-78, 183-186); arrays not supplied start as zeros
  (interp.py:79-81);
* returns a fresh dict holding every declared array.

What changes: the program runs as a hand-written CUDA kernel chosen by the
case discussion evaluated at the live device properties, instead of the
sequential tree walk.  ``tracer`` is CPU-only instrumentation and raises
``NotImplementedError`` (no CPU fallback).  Arrays may be Python lists (as
the reference uses), numpy arrays or torch tensors; results come back in
the same container type.  ``inplace=True`` with contiguous CUDA tensors runs
on the caller's device buffers without copies.
"""

from __future__ import annotations

import threading
import warnings
from dataclasses import dataclass

import numpy as np

from . import _lib, binding, cases, marshal
from .programs import FAMILIES, c_div, effective_params, identify

_INT32_MIN, _INT32_MAX = -(2**31), 2**31 - 1


@dataclass
class RunInfo:
    """What the last run_program call executed (for tests and reports)."""

    family: str
    case: int | None
    applied: tuple[str, ...]
    fallback: bool
    launch: dict
    footprint_words: int


_last: RunInfo | None = None


def last_run() -> RunInfo | None:
    return _last


def _torch():
    import torch

    return torch


def _kind_of(value) -> str:
    if isinstance(value, np.ndarray):
        return "numpy"
    if type(value).__module__.startswith("torch"):
        return "torch"
    return "list"


def _numel(shape) -> int:
    n = 1
    for d in shape:
        n *= d
    return n


def _to_device_tensor(name, value, shape, np_dtype, device):
    """int32 device copy of a caller's array for the emitted-leaf path
    (jit.run_program_jit): IndexError when shorter than declared,
    OverflowError outside int32 (the emitted leaves are C-int kernels)."""
    torch = _torch()
    k = _kind_of(value)
    want = _numel(shape)
    if k == "torch":
        t = value.detach()
        if t.numel() < want:
            raise IndexError("array %s has %d elements; the program declares %s" % (name, t.numel(), shape))
        if np_dtype == np.int32 and t.dtype != torch.int32:
            if t.is_floating_point():
                raise TypeError("array %s: float data for an int program" % name)
            t64 = t.to(torch.int64)
            if t64.numel() and (int(t64.min()) < _INT32_MIN or int(t64.max()) > _INT32_MAX):
                raise OverflowError("array %s holds values outside int32" % name)
            t = t64.to(torch.int32)
        elif np_dtype == np.float32 and t.dtype != torch.float32:
            t = t.to(torch.float32)
        return t.reshape(-1).to(device, copy=True).contiguous(), t.numel()
    if k == "list":
        arr = np.asarray(value, dtype=np.float64 if np_dtype == np.float32 else object)
        if np_dtype == np.int32:
            flat = arr.reshape(-1)
            if flat.size and (min(flat) < _INT32_MIN or max(flat) > _INT32_MAX):
                raise OverflowError("array %s holds values outside int32" % name)
        arr = arr.astype(np_dtype)
    else:
        arr = value
        if np_dtype == np.int32 and arr.dtype != np.int32:
            if np.issubdtype(arr.dtype, np.floating):
                raise TypeError("array %s: float data for an int program" % name)
            if arr.size and (arr.min() < _INT32_MIN or arr.max() > _INT32_MAX):
                raise OverflowError("array %s holds values outside int32" % name)
        arr = np.ascontiguousarray(arr, dtype=np_dtype)
    flat = arr.reshape(-1)
    if flat.size < want:
        raise IndexError("array %s has %d elements; the program declares %s" % (name, flat.size, shape))
    host = torch.from_numpy(flat)
    return host.to(device, non_blocking=False), flat.size


def _shapes_py(fam, P):
    """Array extents with the interpreter's list semantics ([0]*negative == [])."""
    out = {}
    for name, dims in fam.shapes(P).items():
        out[name] = tuple(max(0, d) for d in dims)
    return out


class _PinnedPool:
    """Page-locked staging buffers for the host-array path, kept across calls
    (pinning is slow; pk_run_host needs pinned memory to overlap its PCIe
    copies with the kernels).  One set per declared-array slot, grown on
    demand; a lock serialises callers (each call holds its buffers until the
    results are copied out)."""

    def __init__(self):
        import threading

        self.lock = threading.Lock()
        self.bufs: dict[int, object] = {}

    def view(self, slot: int, count: int, dtype) -> np.ndarray:
        torch = _torch()
        nbytes = max(count, 1) * np.dtype(dtype).itemsize
        buf = self.bufs.get(slot)
        if buf is None or buf.numel() < nbytes:
            cap = 1 << max(20, (nbytes - 1).bit_length())  # powers of two, >= 1 MiB
            self.bufs[slot] = None
            buf = torch.empty(cap, dtype=torch.uint8, pin_memory=True)
            self.bufs[slot] = buf
        return buf.numpy()[:nbytes].view(dtype)

    def release(self) -> None:
        self.bufs.clear()


_pinned = _PinnedPool()


def run_program(
    program,
    params: dict,
    arrays: dict | None = None,
    tracer=None,
    *,
    machine=None,
    device=None,
    inplace: bool = False,
    generic: bool = False,
    case: int | None = None,
    tf32x3: bool = False,
    temporal: int = 0,
    devices=None,
    halo: int = 0,
    via_generic: bool = False,
) -> dict:
    """Execute the whole program on the GPU; returns the final array contents.

    Values keep the reference's semantics (marshal.py): Python floats and
    float64 data compute in binary64 with the interpreter's rounding
    sequence, float32 data on the float32 path (FFMA matmul, BASELINE
    configs[0-1]), ints exactly (int32 or int64 words, ``OverflowError``
    beyond int64); reverse / transpose return the very objects they moved.

    Host arrays (lists, numpy, CPU tensors) go through ``pk_run_host`` from
    pooled pinned buffers: uploads, kernels and downloads overlap.  CUDA
    tensors stay on their device (``inplace=True`` runs on them without a
    copy).

    ``machine``: the machine values for case selection (default: the live
    device).  ``case``: force a leaf by index (tests / tuner).  ``generic``:
    force the program's literal thread mapping instead of the tuned tile.
    Optional variants, reported separately from the leaves: ``tf32x3``
    (float32 matmul on tcgen05, fp32-level accuracy) and ``temporal=h``
    (1-D / 2-D Jacobi advancing h steps per HBM pass, bit-identical).
    ``devices=[d0, d1, ...]``: run on several GPUs of this process
    (pk_launch_multi: unit shares, ghost-zone exchange of width ``halo``
    by peer copies for the stencils); the result is gathered on ``d0``.
    ``via_generic``: run the program through the generic path (generic.py:
    any program, our emitted kernel) even when it is one of the families --
    the path programs outside the families take.
    """
    global _last
    if tracer is not None:
        raise NotImplementedError(
            "tracer is CPU-only instrumentation of the reference interpreter; "
            "the GPU executor cannot report per-access events"
        )
    if via_generic:
        kind = None
    else:
        try:
            kind = identify(program)
        except NotImplementedError:
            kind = None
    if kind is None:
        # outside the seven families (or asked for): the generic path -- our
        # parser and CUDA emitter, NVRTC for sm_100a, the interpreter's value
        # semantics (generic.py); no parakern needed
        from . import generic
        from .programs import program_text

        if not via_generic:
            warnings.warn("program matches none of the seven kernel families: running it through the generic "
                          "emitted kernel (no hand-written kernel)", RuntimeWarning, stacklevel=2)
        out = generic.run_program(program_text(program), params, arrays, device=device)
        g = generic.last
        _last = RunInfo("generic", None, (), False, {"mode": g.mode, "flat": g.flat, "launches": g.launches}, 0)
        return out
    rename = dict(kind.rename)
    if rename:  # an alpha-renamed copy of a known program: speak the family's names inside
        params = {rename.get(k, k): v for k, v in params.items()}
        arrays = {rename.get(k, k): v for k, v in (arrays or {}).items()}
    P = effective_params(kind, params)
    fam = FAMILIES[kind.family]
    torch = _torch()
    if not torch.cuda.is_available():
        raise RuntimeError("run_program needs a CUDA device (sm_100a); there is no CPU fallback")
    if devices is not None:
        devices = [int(d) for d in devices]
        if not devices:
            raise ValueError("devices must name at least one GPU")
        device = devices[0]
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)

    arrays = dict(arrays or {})  # arrays the program does not declare come back as copies (below)
    declared = [a.name for a in fam.arrays]
    plan, srcs = marshal.plan(kind.family, P, {n: arrays[n] for n in declared if n in arrays})

    if machine is None or machine == "live":
        from . import machine as machine_mod

        mv = machine_mod.live(dev.index, elem_bytes=plan.elem_bytes)
    else:
        mv = machine

    # case discussion: an original program selects its leaf at the live
    # machine; a case program already is one
    if kind.is_original:
        sel = cases.select(kind, P, mv)
        if case is not None:
            tab = cases.table(kind.family, sel.machine)
            forced = [c for c in tab.cases if c.index == case]
            if not forced:
                raise ValueError("no case %d for %s" % (case, kind.family))
            sel = cases.Selection(kind.family, sel.machine, forced[0], sel.assignment)
        applied, case_index, fallback = sel.applied, sel.index, sel.fallback
    else:
        applied, case_index, fallback = kind.applied, None, False

    shapes = _shapes_py(fam, P)
    counts = {n: _numel(shapes[n]) for n in declared}
    kinds = [marshal.kind_of(v) for v in arrays.values()]
    default_kind = kinds[0] if kinds else "list"

    L = binding.make_launch(kind, P, applied, plan.dtype, generic=generic,
                            extra_flags=(_lib.FLAG_TF32X3 if tf32x3 else 0) | (_lib.FLAG_TEMPORAL if temporal else 0))
    if temporal:
        L.tblock = int(temporal)  # steps fused per HBM pass (odd; Jacobi programs only)
    # IndexError exactly where an access of the run would leave a supplied array
    need = _lib.required_elems(L, len(declared))
    if kind.family == "jacobi" and need[0]:
        # the 1-D program reads up to a[N + P + 1] (jacobi.mfk, t = 0); the C
        # ABI asks for the whole double buffer, which the shim allocates anyway
        tile = P["s"] * P["B"]
        need[0] = P["N"] + max(0, _c_div(P["N"] - 2, tile)) * tile + 2
    for i, n in enumerate(declared):
        if n in srcs and srcs[n].size < need[i]:
            raise IndexError("access %s[%d] out of bounds (size %d)" % (n, need[i] - 1, srcs[n].size))
    runnable = all(counts[n] > 0 for n in declared)
    on_device = any(s.kind == "torch" and s.value.is_cuda for s in srcs.values())
    multi = devices is not None and len(devices) > 1
    words, out, owned = {}, {}, False
    written = set(fam.written)
    if not on_device and not multi and not inplace:
        # host arrays: pk_run_host_io reads the caller's own buffers where they
        # already hold the plan's words (pageable memory is staged inside the
        # pipeline, overlapped with the DMA and the kernels) and writes results
        # into fresh arrays; other inputs are converted into pooled pinned
        # buffers.  While the GPU runs, this thread copies out the arrays the
        # program never writes (the reference deep-copies them, interp.py:183-186).
        owned = True
        copied = {}
        with _pinned.lock:
            ins, outs = [], []
            for i, n in enumerate(declared):
                src = srcs.get(n)
                direct = marshal.direct_words(plan, src, counts[n])
                if direct is not None:
                    ins.append(direct.ctypes.data)
                    keep = direct  # noqa: F841 -- alive until the call returns
                elif src is None and not plan.objects:
                    ins.append(0)  # zeros (interp.py:79-81)
                else:
                    buf = _pinned.view(i, counts[n], plan.np_dtype)
                    marshal.host_words(plan, src, counts[n], buf)
                    ins.append(buf.ctypes.data)
                if n in written:
                    words[n] = marshal.fresh_array(counts[n], plan.np_dtype)
                    outs.append(words[n].ctypes.data)
                elif direct is not None and direct.size == counts[n] > 0 and runnable:
                    # the library copies the input into a fresh array in the pass that stages it
                    copied[n] = marshal.fresh_array(counts[n], direct.dtype)
                    outs.append(copied[n].ctypes.data)
                else:
                    outs.append(0)
            failure = []
            worker = None
            if runnable:
                def work():
                    try:
                        _lib.run_host_io(L, ins, outs, [counts[n] for n in declared], dev.index)
                    except BaseException as exc:  # re-raised on the caller's thread
                        failure.append(exc)

                worker = threading.Thread(target=work, name="pk_run_host")
                worker.start()
            try:
                for n in declared:
                    if n not in written and n not in copied:
                        like = arrays.get(n)
                        k = marshal.kind_of(like) if like is not None else default_kind
                        out[n] = marshal.copy_input(plan, srcs.get(n), shapes[n], k, like)
            finally:
                if worker is not None:
                    worker.join()
            if failure:
                raise failure[0]
            for n, arr in copied.items():
                src = srcs[n]
                like = arrays.get(n)
                k = marshal.kind_of(like)
                arr = arr.view(src.value.dtype) if k == "numpy" else arr
                out[n] = marshal.finish_copy(arr, src, shapes[n], k, like)
            if not runnable:  # nothing ran: the written arrays hold their inputs
                for i, n in enumerate(declared):
                    if n in written:
                        src = srcs.get(n)
                        if src is None and not plan.objects:
                            words[n][:] = 0
                        else:
                            marshal.host_words(plan, src, counts[n], words[n])
    else:
        stream = torch.cuda.current_stream(dev).cuda_stream
        with torch.cuda.device(dev):
            bufs = []
            for n in declared:
                v = arrays.get(n)
                if (inplace and v is not None and marshal.kind_of(v) == "torch" and v.is_cuda and v.is_contiguous()
                        and not plan.objects and v.dtype == marshal.torch_dtype(plan)):
                    t = v.reshape(-1)
                elif n in srcs:
                    t = marshal.device_words(plan, srcs[n], counts[n], dev)
                elif plan.objects:
                    t = torch.full((max(counts[n], 1),), plan.zero_index, dtype=torch.int64, device=dev)
                else:
                    t = torch.zeros(max(counts[n], 1), dtype=marshal.torch_dtype(plan), device=dev)
                bufs.append(t)
            if runnable:
                if multi:
                    # inputs replicated on every device (full-size arrays, global indexing)
                    reps = [bufs] + [[b.to(torch.device("cuda", d), copy=True) for b in bufs] for d in devices[1:]]
                    for d in set(devices):
                        torch.cuda.synchronize(d)
                    _lib.launch_multi(L, devices, [[b.data_ptr() for b in r] for r in reps], halo=halo)
                else:
                    _lib.launch_checked(L, [b.data_ptr() for b in bufs], [b.numel() for b in bufs], stream)
            torch.cuda.current_stream(dev).synchronize()
        for n, t in zip(declared, bufs):
            words[n] = t

    _last = RunInfo(kind.family, case_index, tuple(applied), fallback, binding.describe(L),
                    _lib.footprint_words(L))

    # arrays the caller passed that the program does not declare come back as copies
    for name, v in arrays.items():
        if name not in counts:
            out[name] = _deep_copy(v)
    for n in declared:
        if n in out:
            continue
        like = arrays.get(n)
        if (inplace and like is not None and marshal.kind_of(like) == "torch" and like.is_cuda
                and words[n].data_ptr() == like.data_ptr()):
            out[n] = like
            continue
        k = marshal.kind_of(like) if like is not None else default_kind
        out[n] = marshal.finish(plan, srcs.get(n), words[n], shapes[n], k, like, owned=owned)
    if rename:
        back = {v: k for k, v in rename.items()}
        out = {back.get(k, k): v for k, v in out.items()}
    return out


def _deep_copy(v):
    if isinstance(v, list):
        return [row[:] if isinstance(row, list) else row for row in v]
    if isinstance(v, np.ndarray):
        return v.copy()
    return v.clone()


# grid meta_for variables (outer first) and the serial context loop of each family's program
GRID_VARS = {"reverse": ("i",), "transpose": ("v0", "v1"), "jacobi": ("i",), "jacobi2d": ("v0", "v1"),
             "matvec": ("i",), "matmul": ("i", "j"), "addition": ("v0", "v1")}
CONTEXT_VARS = {"jacobi": ("t",), "jacobi2d": ("t",), "matmul": ("k",)}


def _block_accesses(family: str, P: dict, g: tuple, ctx: tuple) -> dict:
    """Every index one thread block touches, per array and dimension, as
    (min, max) -- the thread loops and serial loops enumerated exactly (the
    block's accesses are what interp.py:209-212 bounds-checks).  Empty
    dict when the thread loops are empty (nothing runs)."""
    ar = np.arange

    def grid(*ranges):
        mesh = np.meshgrid(*[ar(r, dtype=np.int64) for r in ranges], indexing="ij")
        return [m.reshape(-1) for m in mesh]

    def mm(x):
        return (int(x.min()), int(x.max()))

    N = P["n"] if family == "matmul" else P["N"]
    s = P.get("s", 1)
    if family in ("reverse", "jacobi", "matvec"):
        j, k = grid(max(0, P["B"]), max(0, s))
        if j.size == 0:
            return {}
        p = g[0] * s * P["B"] + k * P["B"] + j
        if family == "reverse":
            return {"a": [mm(p)], "c": [mm(N - 1 - p)]}
        if family == "jacobi":
            src = N + p if ctx[0] % 2 == 0 else p
            dst = p + 1 if ctx[0] % 2 == 0 else N + p + 1
            return {"a": [(min(int(src.min()), int(dst.min())), max(int(src.max()) + 2, int(dst.max())))]}
        if N <= 0:  # the q loop is empty: the statement never runs
            return {}
        return {"a": [mm(p), (0, N - 1)], "x": [(0, N - 1)], "y": [mm(p)]}
    if family == "matmul":
        v, u, w = grid(max(0, P["B0"]), max(0, P["ub1"]), max(0, s))
        if v.size == 0:
            return {}
        p = g[0] * P["B0"] + v
        q = g[1] * P["ub1"] * s + w * P["ub1"] + u
        out = {"c": [mm(p), mm(q)]}
        if P["B0"] > 0:
            kk = (P["B0"] * ctx[0], P["B0"] * ctx[0] + P["B0"] - 1)
            out["a"] = [mm(p), kk]
            out["b"] = [kk, mm(q)]
        return out
    u0, u1, k = grid(max(0, P["B0"]), max(0, P["B1"]), max(0, s if family != "addition" else 1))
    if u0.size == 0:
        return {}
    if family == "transpose":
        i = g[0] * P["B0"] + u0
        jj = (g[1] * s + k) * P["B1"] + u1
        return {"a": [mm(jj), mm(i)], "c": [mm(i * N + jj)]}
    if family == "jacobi2d":
        i = g[0] * P["B0"] + u0 + 1
        jj = (g[1] * s + k) * P["B1"] + u1 + 1
        rows = [int(i.min()) - 1, int(i.max()) + 1]
        if ctx[0] % 2 == 0:
            return {"a": [(rows[0], N + int(i.max())), (int(jj.min()) - 1, int(jj.max()) + 1)]}
        return {"a": [(int(i.min()), N + rows[1]), (int(jj.min()) - 1, int(jj.max()) + 1)]}
    # addition: the guard i < N && j < N/2 (merged: j < N) selects the points that access
    i = g[0] * P["B0"] + u0
    jj = g[1] * P["B1"] + u1
    merged = P.get("_merged", False)
    keep = (i < N) & (jj < (N if merged else N // 2))
    if not keep.any():
        return {}
    idx = (i * N + jj)[keep]
    hi = int(idx.max()) + (0 if merged else N // 2)
    return {n: [(int(idx.min()), hi)] for n in ("a", "b", "c")}


def run_block(program, params, grid_values, context_values=None, arrays=None, tracer=None):
    """One thread block (interp.py:228-249): the grid indices fixed to
    ``grid_values``, the serial context loop variables to ``context_values``,
    the thread loops swept -- by one CUDA block of the family's block kernel
    (pk_launch_block, csrc/k_block.cu) in the program's own statement order.
    Values follow run_program's rules (marshal.py: binary64 for Python
    floats, int64 where int32 could not hold the values, object words for the
    permutations); an access outside an array raises ``IndexError`` as the
    reference does.  Returns every declared array like run_program."""
    global _last
    if tracer is not None:
        raise NotImplementedError(
            "tracer is CPU-only instrumentation of the reference interpreter; "
            "the GPU executor cannot report per-access events"
        )
    try:
        kind = identify(program)
    except NotImplementedError:
        # outside the seven families: one block of the generic path's kernel
        from . import generic
        from .programs import program_text

        out = generic.run_block(program_text(program), params, grid_values, context_values, arrays)
        g = generic.last
        _last = RunInfo("generic", None, (), False, {"mode": g.mode, "block": True, "launches": g.launches}, 0)
        return out
    rename = dict(kind.rename)
    grid_values = {rename.get(k, k): v for k, v in dict(grid_values).items()}
    context_values = {rename.get(k, k): v for k, v in dict(context_values or {}).items()}
    params = {rename.get(k, k): v for k, v in params.items()}
    arrays = {rename.get(k, k): v for k, v in dict(arrays or {}).items()}
    fam = FAMILIES[kind.family]
    P = effective_params(kind, params)
    g = []
    for name in GRID_VARS[kind.family]:
        if name not in grid_values:
            raise KeyError(name)  # the body reads the grid variable (interp.py eval of an unset Name)
        g.append(int(grid_values[name]))
    ctx = []
    for name in CONTEXT_VARS.get(kind.family, ()):
        if name not in context_values:
            raise KeyError(name)
        ctx.append(int(context_values[name]))
    torch = _torch()
    if not torch.cuda.is_available():
        raise RuntimeError("run_block needs a CUDA device (sm_100a); there is no CPU fallback")
    declared = [a.name for a in fam.arrays]
    plan, srcs = marshal.plan(kind.family, P, {n: arrays[n] for n in declared if n in arrays})
    shapes = _shapes_py(fam, P)
    merged = kind.family == "addition" and "granularity" in kind.applied
    acc = _block_accesses(kind.family, dict(P, _merged=merged), tuple(g), tuple(ctx))
    for name, dims in acc.items():
        shape = tuple(np.shape(np.asarray(arrays[name], dtype=object))) if name in arrays and \
            marshal.kind_of(arrays[name]) == "list" else \
            (tuple(arrays[name].shape) if name in arrays else shapes[name])
        if len(shape) != len(dims):  # flat data for a 2-D declaration: check the flat extent
            shape, dims = (int(np.prod(shape)),), [(dims[0][0] * shapes[name][-1] + dims[-1][0],
                                                    dims[0][1] * shapes[name][-1] + dims[-1][1])]
        for (lo, hi), n in zip(dims, shape):
            if lo < 0 or hi >= n:
                raise IndexError("access %s out of bounds: index %d, size %d" % (name, lo if lo < 0 else hi, n))
    dev = torch.device("cuda", torch.cuda.current_device())
    counts = {n: _numel(shapes[n]) for n in declared}
    bufs = []
    for n in declared:
        if n in srcs:
            bufs.append(marshal.device_words(plan, srcs[n], counts[n], dev))
        elif plan.objects:
            bufs.append(torch.full((max(counts[n], 1),), plan.zero_index, dtype=torch.int64, device=dev))
        else:
            bufs.append(torch.zeros(max(counts[n], 1), dtype=marshal.torch_dtype(plan), device=dev))
    L = binding.make_launch(kind, P, kind.applied, plan.dtype)
    if acc and all(counts[n] > 0 for n in declared):
        _lib.launch_block(L, g, ctx, [b.data_ptr() for b in bufs], torch.cuda.current_stream(dev).cuda_stream)
    torch.cuda.current_stream(dev).synchronize()
    _last = RunInfo(kind.family, None, tuple(kind.applied), False,
                    dict(binding.describe(L), block=True, grid=g, context=ctx), 0)
    kinds = [marshal.kind_of(v) for v in arrays.values()]
    default_kind = kinds[0] if kinds else "list"
    out = {}
    for name, v in arrays.items():
        if name not in counts:
            out[name] = _deep_copy(v)
    for n, t in zip(declared, bufs):
        like = arrays.get(n)
        k = marshal.kind_of(like) if like is not None else default_kind
        out[n] = marshal.finish(plan, srcs.get(n), t, shapes[n], k, like)
    if rename:
        back = {v: k for k, v in rename.items()}
        out = {back.get(k, k): v for k, v in out.items()}
    return out


_c_div = c_div  # interp.py:43-46, defined once in programs.py


def c_mod(a: int, b: int) -> int:
    """C99 remainder (interp.py:49-50)."""
    return a - b * c_div(a, b)
