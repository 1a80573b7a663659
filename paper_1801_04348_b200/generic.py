"""GPU path for ``.mfk`` programs outside the seven hand-written kernel
families -- self-contained: our own parser (mfk.py), our own CUDA emitter,
NVRTC for sm_100a, no parakern at run time.

SURVEY 8(f) row 2.  ``run_program`` (interp.py) routes a program here when
its token stream is none of the families'.  Semantics are the reference
interpreter's (/root/reference/pkg/src/parakern/interp.py):

* declarations in order (interp.py:62-81): bindings evaluated with C
  division, array extents, a ``KeyError`` for the first declared scalar
  without a value; caller arrays copied, undeclared ones zero-filled; every
  array (declared or supplied) comes back in a fresh dict;
* the serial context loops run on the host, one kernel launch per iteration
  (interp.py:140-145); the meta_for nest runs in parallel -- the language
  guarantees no dependence between its iterations within one pass
  (interp.py:12-15), which is what makes the parallel schedule equal the
  sequential walk;
* values: ints exact (int64 words; ``OverflowError`` where the reference's
  unbounded ints leave int64), Python floats binary64 with the
  interpreter's rounding sequence, ``/`` and ``%`` as c_div / c_mod on ints
  and on floats (CPython float floor division of the absolute values),
  bools and any other objects moved unchanged (pk_generic_rt.cuh);
* errors as the reference: ``IndexError`` out of bounds (per subscript,
  against the caller's lengths), ``ZeroDivisionError``, ``TypeError`` (float
  subscripts, arithmetic on objects), ``KeyError`` (missing parameter,
  undeclared name or array).  When several iterations fail, the exception
  raised is the first one recorded on the device, not necessarily the
  sequentially first.

Mapping: when every meta_for bound depends only on parameters, bindings and
context variables (a rectangular nest) the whole nest is flattened into one
grid-stride loop of 256-thread blocks, innermost variable fastest (so
consecutive threads touch consecutive elements for the usual programs);
otherwise the grid / thread roles of the nest (dsl.split_roles) map onto
grid-stride loops over blockIdx / threadIdx.
"""

from __future__ import annotations

import os
import threading
from dataclasses import dataclass

import numpy as np

from . import _lib, mfk

_I64_MIN, _I64_MAX = -(2**63), 2**63 - 1
_RT_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "csrc", "pk_generic_rt.cuh")
_CMP = {"<": 0, "<=": 1, ">": 2, ">=": 3, "==": 4, "!=": 5}
_OPS = {"+": "v_add", "-": "v_sub", "*": "v_mul", "/": "v_div", "%": "v_mod"}
_ERR = {1: IndexError, 2: ZeroDivisionError, 3: OverflowError, 4: TypeError, 5: KeyError}

T_INT, T_FLOAT, T_BOOL, T_OBJ = 0, 1, 2, 3


def c_div(a, b):
    """interp.py:43-46 on Python numbers (ints and floats alike)."""
    q = abs(a) // abs(b)
    return q if (a >= 0) == (b >= 0) else -q


def c_mod(a, b):
    return a - b * c_div(a, b)


# ---------------------------------------------------------------- host eval --

def host_eval(e, env: dict):
    """An expression over scalars on the host (bindings, extents, context and
    rectangular meta bounds); array reads are not available here."""
    k = e[0]
    if k == "num":
        return e[1]
    if k == "name":
        if e[1] not in env:
            raise KeyError(e[1])
        return env[e[1]]
    if k == "bin":
        a, b = host_eval(e[2], env), host_eval(e[3], env)
        op = e[1]
        if op == "+":
            return a + b
        if op == "-":
            return a - b
        if op == "*":
            return a * b
        if op == "/":
            return c_div(a, b)
        return c_mod(a, b)
    raise KeyError(e[1])  # an array read while the arrays do not exist yet (interp.py:62-71)


def _names(e) -> set:
    return {n[1] for n in mfk.walk_exprs(e) if n[0] == "name"}


def _has_index(e) -> bool:
    return any(n[0] == "idx" for n in mfk.walk_exprs(e))


# ------------------------------------------------------------------ arrays --

@dataclass
class HostArray:
    name: str
    rank: int
    rows: int
    cols: int
    kind: str                 # list | numpy | torch | zeros
    like: object = None       # the caller's array (dtype / device for the result)
    flat: list | None = None  # list input: flat Python values
    np_flat: np.ndarray | None = None  # numpy / torch input: flat values


def _host_array(name: str, value) -> HostArray:
    if isinstance(value, np.ndarray) or type(value).__module__.startswith("torch"):
        kind = "numpy" if isinstance(value, np.ndarray) else "torch"
        a = value if kind == "numpy" else value.detach().cpu().numpy()
        if a.ndim not in (1, 2):
            raise NotImplementedError("array %r: %d dimensions (the language has 1 or 2)" % (name, a.ndim))
        rows, cols = (a.shape[0], a.shape[1] if a.ndim == 2 else 0)
        return HostArray(name, a.ndim, rows, cols, kind, value, np_flat=np.ascontiguousarray(a).reshape(-1))
    value = list(value)
    if value and isinstance(value[0], list):  # the reference's 2-D test (interp.py:183-186)
        cols = len(value[0])
        if any(not isinstance(r, list) or len(r) != cols for r in value):
            raise NotImplementedError("array %r: ragged 2-D list" % name)
        return HostArray(name, 2, len(value), cols, "list", value, flat=[v for r in value for v in r])
    return HostArray(name, 1, len(value), 0, "list", value, flat=value)


def _all_int(h: HostArray) -> bool:
    if h.np_flat is not None:
        a = h.np_flat
        if a.dtype.kind == "i":
            return True
        if a.dtype.kind == "u":
            return a.size == 0 or int(a.max()) <= _I64_MAX
        return False
    return all(type(v) is int and _I64_MIN <= v <= _I64_MAX for v in h.flat)


def _encode_dyn(h: HostArray, pool: list) -> np.ndarray:
    """(n, 2) int64: value bits, tag."""
    n = h.rows * (h.cols if h.rank == 2 else 1)
    out = np.zeros((n, 2), dtype=np.int64)
    if h.np_flat is not None and h.np_flat.dtype.kind in "iub":
        a = h.np_flat
        if a.dtype.kind == "u" and a.size and int(a.max()) > _I64_MAX:
            raise OverflowError("array %r: values beyond int64" % h.name)
        out[:, 0] = a.astype(np.int64)
        out[:, 1] = T_BOOL if a.dtype.kind == "b" else T_INT
        return out
    if h.np_flat is not None and h.np_flat.dtype.kind == "f":
        out[:, 0] = h.np_flat.astype(np.float64).view(np.int64)
        out[:, 1] = T_FLOAT
        return out
    vals = h.flat if h.flat is not None else h.np_flat.tolist()
    for k, v in enumerate(vals):
        t = type(v)
        if t is int:
            if not _I64_MIN <= v <= _I64_MAX:
                raise OverflowError("array %r: %d does not fit int64" % (h.name, v))
            out[k] = (v, T_INT)
        elif t is float:
            out[k, 0] = np.array(v, dtype=np.float64).view(np.int64)
            out[k, 1] = T_FLOAT
        elif t is bool:
            out[k] = (int(v), T_BOOL)
        else:
            out[k] = (len(pool), T_OBJ)
            pool.append(v)
    return out


def _decode(h: HostArray, words: np.ndarray, mode: str, pool: list, container: str):
    """Device words -> the caller's container (a fresh object)."""
    n = words.shape[0]
    if mode in ("int", "int32"):
        vals = words
        if container == "list":
            flat = vals.tolist()
        else:
            dt = h.like.dtype if h.like is not None and hasattr(h.like, "dtype") else np.dtype(np.int64)
            dt = np.dtype(str(dt).replace("torch.", "")) if not isinstance(dt, np.dtype) else dt
            if dt.kind in "iu" and n and (vals.min() < np.iinfo(dt).min or vals.max() > np.iinfo(dt).max):
                dt = np.dtype(np.int64)
            flat = vals.astype(dt if dt.kind in "iu" else np.int64)
    else:
        bits, tags = words[:, 0], words[:, 1]
        if container == "list":
            flat = [None] * n
            fl = bits.view(np.float64)
            for k in range(n):
                t = tags[k]
                flat[k] = (int(bits[k]) if t == T_INT else float(fl[k]) if t == T_FLOAT
                           else bool(bits[k]) if t == T_BOOL else pool[int(bits[k])])
        else:
            like_dt = getattr(h.like, "dtype", None)
            like_dt = np.dtype(str(like_dt).replace("torch.", "")) if like_dt is not None and not isinstance(
                like_dt, np.dtype) else like_dt
            if (tags == T_OBJ).any():
                flat = np.array([pool[int(b)] if t == T_OBJ else (float(np.int64(b).view(np.float64)) if t == T_FLOAT
                                 else bool(b) if t == T_BOOL else int(b)) for b, t in zip(bits, tags)], dtype=object)
            elif (tags == T_FLOAT).any():
                f = np.where(tags == T_FLOAT, bits.view(np.float64), bits.astype(np.float64))
                flat = f.astype(like_dt if like_dt is not None and like_dt.kind == "f" else np.float64)
            elif n and (tags == T_BOOL).all() and like_dt is not None and like_dt.kind == "b":
                flat = bits.astype(bool)
            else:
                dt = like_dt if like_dt is not None and like_dt.kind in "iu" else np.dtype(np.int64)
                if n and (bits.min() < np.iinfo(dt).min or bits.max() > np.iinfo(dt).max):
                    dt = np.dtype(np.int64)
                flat = bits.astype(dt)
    if container == "list":
        if h.rank == 2:
            return [flat[r * h.cols:(r + 1) * h.cols] for r in range(h.rows)]
        return flat
    arr = flat.reshape((h.rows, h.cols) if h.rank == 2 else (h.rows,))
    if container == "torch":
        import torch

        t = torch.from_numpy(np.ascontiguousarray(arr)) if arr.dtype != object else arr
        dev = getattr(h.like, "device", None)
        return t.to(dev) if dev is not None and hasattr(t, "to") else t
    return arr


# ----------------------------------------------------------------- emitter --

class _Emitter:
    """CUDA text of one program for one value model."""

    def __init__(self, prog: mfk.Program, mode: str, env_names: list, array_ids: dict, ranks: dict,
                 flat: bool):
        self.p, self.mode, self.env, self.ids, self.ranks, self.flat = prog, mode, env_names, array_ids, ranks, flat
        self.lines: list[str] = []
        self.n = 0
        self.depth = 1
        # every scalar name the kernel may read or write: the program's flat environment
        names = set(env_names)
        for var, _, _ in prog.meta:
            names.add(var)
        for s in mfk.walk_exprs(prog.body):
            if s[0] == "name":
                names.add(s[1])
        for var, bound, _ in prog.meta:
            names |= _names(bound)

        def stmt_names(stmts):
            for s in stmts:
                if s[0] == "local":
                    names.add(s[1])
                elif s[0] == "assign" and s[1][0] == "name":
                    names.add(s[1][1])
                elif s[0] == "for":
                    names.add(s[1])
                    stmt_names(s[3])
                elif s[0] == "if":
                    stmt_names(s[2])
                    stmt_names(s[3] or ())

        stmt_names(prog.body)
        self.names = sorted(names)
        # names with a value somewhere: the environment, the meta variables and
        # whatever the body assigns; any other name raises KeyError when read
        assigned = set()

        def assigned_in(stmts):
            for s in stmts:
                if s[0] == "local":
                    assigned.add(s[1])
                elif s[0] == "assign" and s[1][0] == "name":
                    assigned.add(s[1][1])
                elif s[0] == "for":
                    assigned.add(s[1])
                    assigned_in(s[3])
                elif s[0] == "if":
                    assigned_in(s[2])
                    assigned_in(s[3] or ())

        assigned_in(prog.body)
        self.defined = set(env_names) | {v for v, _, _ in prog.meta} | assigned

    def w(self, text: str) -> None:
        self.lines.append("    " * self.depth + text)

    def tmp(self) -> str:
        self.n += 1
        return "t%d" % self.n

    def var(self, name: str) -> str:
        return "s_" + name

    # expressions: emitted as one temporary per node, left to right (Python's order)
    def ex(self, e) -> str:
        k = e[0]
        t = self.tmp()
        if k == "num":
            if not _I64_MIN <= e[1] <= _I64_MAX:
                raise OverflowError("literal %d does not fit int64" % e[1])
            self.w("const V %s = PK_LIT(%dLL);" % (t, e[1]) if e[1] != _I64_MIN else
                   "const V %s = PK_LIT((-9223372036854775807LL - 1));" % t)
        elif k == "name":
            if e[1] in self.defined:
                self.w("const V %s = v_def(err, %s);" % (t, self.var(e[1])))
            else:
                self.w("pk_fail(err, PK_E_KEY, -2, 0, 0);")
                self.w("const V %s = PK_ZERO;" % t)
        elif k == "bin":
            a, b = self.ex(e[2]), self.ex(e[3])
            self.w("const V %s = %s(err, %s, %s);" % (t, _OPS[e[1]], a, b))
        else:
            i0, i1 = self.subs(e)
            if i0 is None:
                self.w("const V %s = PK_ZERO;" % t)
            else:
                aid = self.ids[e[1]]
                self.w("const V %s = pk_ld(err, %d, A%d, %s, %s, %d);" % (t, aid, aid, i0, i1, self.ranks[e[1]]))
        return t

    def subs(self, e):
        """Subscripts of an array access as i64 temporaries; (None, None) when
        the access fails whatever the indices (an unknown array: KeyError; a
        subscript count that is not the array's rank: TypeError)."""
        name, subs = e[1], e[2]
        if name not in self.ids:
            for s in subs:
                self.ex(s)
            self.w("pk_fail(err, PK_E_KEY, -1, 0, 0);")
            return None, None
        idx = []
        for s in subs:
            v = self.ex(s)
            t = self.tmp()
            self.w("const i64 %s = v_index(err, %s);" % (t, v))
            idx.append(t)
        if len(subs) != self.ranks[name]:
            self.w("pk_fail(err, PK_E_TYPE, 3, 0, 0);")
            return None, None
        return idx[0], (idx[1] if len(idx) > 1 else "0")

    def cond(self, c) -> str:
        t = self.tmp()
        if c[0] == "cmp":
            a, b = self.ex(c[2]), self.ex(c[3])
            self.w("const bool %s = v_cmp(err, %d, %s, %s);" % (t, _CMP[c[1]], a, b))
            return t
        self.w("bool %s = false;" % t)  # &&: short-circuit, as all() over a generator
        opened = 0
        for k, part in enumerate(c[1]):
            r = self.cond(part)
            if k + 1 < len(c[1]):
                self.w("if (%s) {" % r)
                self.depth += 1
                opened += 1
            else:
                self.w("%s = %s;" % (t, r))
        for _ in range(opened):
            self.depth -= 1
            self.w("}")
        return t

    def stmts(self, stmts) -> None:
        for s in stmts:
            k = s[0]
            if k == "local":
                v = self.ex(s[2])
                self.w("%s = %s;" % (self.var(s[1]), v))
            elif k == "assign":
                v = self.ex(s[2])  # the value first, then the subscripts (interp.py:121-127)
                if s[1][0] == "name":
                    self.w("%s = %s;" % (self.var(s[1][1]), v))
                else:
                    i0, i1 = self.subs(s[1])
                    if i0 is not None:
                        aid = self.ids[s[1][1]]
                        self.w("pk_st(err, %d, A%d, %s, %s, %d, v_def(err, %s));"
                               % (aid, aid, i0, i1, self.ranks[s[1][1]], v))
            elif k == "if":
                c = self.cond(s[1])
                self.w("if (%s) {" % c)
                self.depth += 1
                self.stmts(s[2])
                self.depth -= 1
                if s[3] is not None:
                    self.w("} else {")
                    self.depth += 1
                    self.stmts(s[3])
                    self.depth -= 1
                self.w("}")
            else:  # serial for: range(bound), the variable keeps its last value
                b = self.ex(s[2])
                n, q = self.tmp(), self.tmp()
                self.w("const i64 %s = v_bound(err, %s);" % (n, b))
                self.w("for (i64 %s = 0; %s < %s; %s++) {" % (q, q, n, q))
                self.depth += 1
                self.w("if (*(volatile int *)&err->code) return;")
                self.w("%s = vi(%s);" % (self.var(s[1]), q))
                self.stmts(s[3])
                self.depth -= 1
                self.w("}")

    def kernel(self) -> str:
        p = self.p
        self.w("const int pk_unused = 0; (void)pk_unused;")
        for aid in range(len(self.ids)):
            self.w("const PkArr A%d = arrs[%d];" % (aid, aid))
        for name in self.names:
            if name in self.env:
                self.w("V %s = vi(frame[%d]);" % (self.var(name), self.env.index(name)))
            else:
                self.w("V %s = %s;" % (self.var(name), "vundef()" if self.mode == "dyn" else "PK_ZERO"))
        nenv = len(self.env)
        if self.flat:
            # bounds come in the frame after the environment (host-evaluated, outermost first)
            m = len(p.meta)
            self.w("const i64 pk_total = frame[%d];" % (nenv + m))
            self.w("for (i64 L = (i64)blockIdx.x * blockDim.x + threadIdx.x; L < pk_total; "
                   "L += (i64)gridDim.x * blockDim.x) {")
            self.depth += 1
            self.w("i64 r = L;")
            for k in range(m - 1, -1, -1):
                var = p.meta[k][0]
                if k:
                    self.w("%s = vi(r %% frame[%d]); r /= frame[%d];" % (self.var(var), nenv + k, nenv + k))
                else:
                    self.w("%s = vi(r);" % self.var(var))
            self.stmts(p.body)
            self.depth -= 1
            self.w("}")
        else:
            dims = {}
            for role, loops, base in (("grid", p.grid, "blockIdx"), ("thread", p.thread, "threadIdx")):
                # the first two loops of a role take the y / x axes; further ones
                # (legal text, dsl.split_roles would refuse to map them) run serially
                axes = ["x"] if len(loops) == 1 else ["y", "x"]
                for (var, _, _), ax in zip(loops[:2], axes):
                    dims[var] = (base, "gridDim" if role == "grid" else "blockDim", ax)
            opened = 0
            for var, bound, _ in p.meta:
                b = self.ex(bound)
                n, q = self.tmp(), self.tmp()
                self.w("const i64 %s = v_bound(err, %s);" % (n, b))
                if var in dims:
                    base, stride, ax = dims[var]
                    self.w("for (i64 %s = %s.%s; %s < %s; %s += %s.%s) {" % (q, base, ax, q, n, q, stride, ax))
                else:
                    self.w("for (i64 %s = 0; %s < %s; %s++) {" % (q, q, n, q))
                self.depth += 1
                self.w("%s = vi(%s);" % (self.var(var), q))
                opened += 1
            self.stmts(p.body)
            for _ in range(opened):
                self.depth -= 1
                self.w("}")
        body = "\n".join(self.lines)
        head = {"int": "#define PK_MODE_INT\n", "int32": "#define PK_MODE_INT\n#define PK_WORD32\n"}.get(self.mode, "")
        with open(_RT_PATH) as fh:
            rt = fh.read()
        return (head + rt + "\n\nextern \"C\" __global__ void __launch_bounds__(1024) pk_generic("
                "const i64 *__restrict__ frame, const PkArr *__restrict__ arrs, PkErr *err) {\n" + body + "\n}\n")


_compiled: dict = {}


def _kernel(source: str) -> int:
    h = _compiled.get(source)
    if h is None:
        h = _lib.jit_compile(source, "pk_generic", ["-DNDEBUG"])
        _compiled[source] = h
    return h


# ---------------------------------------------------------------- runner ---

@dataclass
class GenericRun:
    """What the last generic run did (tests and reports)."""

    mode: str
    flat: bool
    launches: int
    source: str


last: GenericRun | None = None


def _written(prog: mfk.Program) -> set:
    """Arrays the body assigns to (the others come back as host copies)."""
    out = set()

    def walk(stmts):
        for st in stmts:
            if st[0] == "assign" and st[1][0] == "idx":
                out.add(st[1][1])
            elif st[0] == "if":
                walk(st[2])
                walk(st[3] or ())
            elif st[0] == "for":
                walk(st[3])

    walk(prog.body)
    return out


def _fits32(h: HostArray) -> bool:
    if h.kind == "zeros":
        return True
    if h.np_flat is not None:
        a = h.np_flat
        if a.dtype.kind in "iu" and a.dtype.itemsize <= 4 and not (a.dtype.kind == "u" and a.dtype.itemsize == 4):
            return True
        return a.dtype.kind in "iu" and (a.size == 0 or (int(a.min()) >= -2**31 and int(a.max()) < 2**31))
    return all(-2**31 <= v < 2**31 for v in h.flat)


def _host_copy(h: HostArray, container: str):
    """An array the program never writes: a fresh copy of the caller's, as the
    reference returns it (interp.py:76-78), without a device round trip."""
    if h.kind == "list":
        return [r[:] for r in h.like] if h.rank == 2 else list(h.like)
    if h.kind == "numpy":
        return h.like.copy()
    if h.kind == "torch":
        return h.like.clone()
    # declared, not supplied, never written: zeros (interp.py:79-81)
    if container == "list":
        return [[0] * h.cols for _ in range(h.rows)] if h.rank == 2 else [0] * h.rows
    z = np.zeros((h.rows, h.cols) if h.rank == 2 else (h.rows,), dtype=np.int64)
    if container == "torch":
        import torch

        return torch.from_numpy(z)
    return z


_pinned: dict = {}
_lock = threading.Lock()


def _pinned_buffer(nbytes: int):
    """A recycled pinned host buffer (downloads land there at full PCIe speed;
    the results are then converted out of it into fresh arrays)."""
    import torch

    buf = _pinned.get("d2h")
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, pin_memory=True)
        _pinned["d2h"] = buf
    return buf


def run_program(program_text: str, params: dict, arrays: dict | None = None, *, device=None) -> dict:
    """interp.run_program for any parsed program, on the GPU (see the module doc)."""
    return _run(mfk.parse(program_text), params, arrays, device, None)


def run_block(program_text: str, params: dict, grid_values: dict, context_values: dict | None = None,
              arrays: dict | None = None, *, device=None) -> dict:
    """interp.run_block (interp.py:228-249) for any parsed program: the
    declarations with ``params``, then the context and grid values set, then
    the thread loops swept (the grid loops are not run); an access outside an
    array raises IndexError, a name without a value KeyError."""
    import copy

    prog = mfk.parse(program_text)
    if len(prog.grid) > 2 or len(prog.thread) > 2:  # dsl.split_roles (dsl.py:651-656)
        raise mfk.MfkError("at most two grid and two thread dimensions are supported (got %d grid, %d thread)"
                           % (len(prog.grid), len(prog.thread)))
    block = copy.copy(prog)
    block.meta, block.grid, block.thread, block.context = list(prog.thread), [], list(prog.thread), []
    extra = dict(context_values or {})
    extra.update(grid_values)
    return _run(block, params, arrays, device, extra)


def _run(prog: mfk.Program, params: dict, arrays, device, extra) -> dict:
    global last
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("run_program needs a CUDA device (sm_100a); there is no CPU fallback")
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else int(device))

    # declarations in order (interp.py:62-75)
    env = dict(params)
    dims = {}
    for kind, name in prog.decl_order:
        if kind == "binding":
            env[name] = host_eval(dict(prog.bindings)[name], env)
        elif kind == "array":
            dims[name] = tuple(host_eval(d, env) for d in prog.arrays[name])
        elif name not in env:
            raise KeyError("no value supplied for parameter %r" % name)
    if extra:  # run_block: context and grid values after the declarations (interp.py:244-245)
        env.update(extra)
    used = set(prog.scalars) | {b for b, _ in prog.bindings}
    for e in mfk.walk_exprs((prog.body, tuple(b for _, b, _ in prog.meta), tuple(b for _, b in prog.context))):
        if e[0] == "name":
            used.add(e[1])
    env = {k: v for k, v in env.items() if k in used}  # parameters the program never names play no part
    for k, v in list(env.items()):
        if type(v) is bool:
            env[k] = int(v)
        elif type(v) is not int:
            raise TypeError("parameter %r: the GPU path takes int parameters (got %r)" % (k, type(v).__name__))
        if not _I64_MIN <= env[k] <= _I64_MAX:
            raise OverflowError("parameter %r = %d does not fit int64" % (k, env[k]))

    arrays = arrays or {}
    hosts: dict[str, HostArray] = {}
    for name, value in arrays.items():  # caller arrays, declared or not (interp.py:76-78)
        hosts[name] = _host_array(name, value)
    for name, d in dims.items():  # declared arrays not supplied start as zeros (interp.py:79-81)
        if name not in hosts:
            rows = max(d[0], 0)
            hosts[name] = HostArray(name, len(d), rows, max(d[1], 0) if len(d) == 2 and rows else 0, "zeros")
    container = "numpy" if any(h.kind == "numpy" for h in hosts.values()) else (
        "torch" if any(h.kind == "torch" for h in hosts.values()) else "list")
    if all(h.kind == "zeros" or _all_int(h) for h in hosts.values()):
        mode = "int32" if all(_fits32(h) for h in hosts.values()) else "int"
    else:
        mode = "dyn"

    # the environment the kernel starts from: parameters (every one the program
    # names, as the reference's env), bindings, context variables
    ctx_vars = [v for v, _ in prog.context]
    env_names = list(dict.fromkeys(sorted(k for k in env if k not in ctx_vars) + ctx_vars))

    # context iterations on the host (interp.py:140-145), one frame each
    frames = []

    def ctx(k, e):
        if k == len(prog.context):
            frames.append(dict(e))
            return
        var, bound = prog.context[k]
        if _has_index(bound):
            raise NotImplementedError("a context-loop bound that reads an array")
        for v in range(host_eval(bound, e)):
            e2 = dict(e)
            e2[var] = v
            ctx(k + 1, e2)

    ctx(0, env)

    # rectangular nest: every meta bound from the environment only -> flattened
    meta_vars = {v for v, _, _ in prog.meta}
    flat = all(not _has_index(b) and not (_names(b) & meta_vars) and _names(b) <= set(env_names)
               for _, b, _ in prog.meta)
    rows, plans = [], []
    for f in frames:
        vals = [f[k] for k in env_names]
        if flat:
            bounds, total = [], 1
            for _, b, _ in prog.meta:  # outermost first; an empty loop stops the walk (range(<=0))
                v = host_eval(b, f)
                bounds.append(v)
                if v <= 0:
                    total = 0
                    break
                total *= v
            bounds += [1] * (len(prog.meta) - len(bounds))
            if total > _I64_MAX:
                raise OverflowError("meta_for nest of %d iterations" % total)
            vals += bounds + [total]
            plans.append(None if total == 0 else ([min((total + 255) // 256, 148 * 64)], [256]))
        else:
            plans.append((_dims(prog.grid[:2], f, 65535, limit_total=None),
                          _dims(prog.thread[:2], f, 1024, limit_total=1024)))
        rows.append(vals)

    names = list(hosts)
    written = _written(prog)
    while True:  # (the pinned download buffer is shared: one run at a time)
        with _lock:
            out, code, e, src, launches, pool = _execute(prog, mode, hosts, names, written, env_names, rows, plans,
                                                         flat, container, dev)
        if code == 6 and mode == "int32":  # a value left the 32-bit words: again on 64-bit words
            mode = "int"
            continue
        break
    last = GenericRun(mode, flat, launches, src)
    if code:
        exc = _ERR.get(code, RuntimeError)
        if exc is IndexError and 0 <= e[1] < len(names):
            raise IndexError("access %s[%d]%s out of bounds" % (names[e[1]], e[2],
                                                                ("[%d]" % e[3]) if hosts[names[e[1]]].rank == 2 else ""))
        raise exc({1: "index out of range", 2: "division by zero", 3: "integer result beyond int64 (the GPU "
                   "path's ints are 64-bit; the reference's are unbounded)", 4: "unsupported operand or subscript "
                   "type", 5: "name or array read before any value was supplied"}.get(code, "error %d" % code))
    return out


def _execute(prog, mode, hosts, names, written, env_names, rows, plans, flat, container, dev):
    """One device run: upload, launches, error word, downloads."""
    import torch

    ids = {n: k for k, n in enumerate(names)}
    ranks = {n: hosts[n].rank for n in names}
    src = _Emitter(prog, mode, env_names, ids, ranks, flat).kernel()
    h = _kernel(src)
    pool: list = []
    wdt = {"int32": np.int32, "int": np.int64}.get(mode)
    bufs = []
    for n in names:
        hh = hosts[n]
        count = hh.rows * (hh.cols if hh.rank == 2 else 1)
        if hh.kind == "zeros":
            t = torch.zeros(max(count, 1) * (2 if mode == "dyn" else 1), dtype=torch.int64 if wdt is not np.int32
                            else torch.int32, device=dev)
        else:
            if mode == "dyn":
                words = _encode_dyn(hh, pool)
            elif hh.np_flat is not None:
                words = hh.np_flat.astype(wdt, copy=False)
            else:
                words = np.array(hh.flat, dtype=wdt) if count else np.zeros(0, wdt)
            t = torch.from_numpy(np.ascontiguousarray(words)).to(dev, non_blocking=False)
            if t.numel() == 0:
                t = torch.zeros(2, dtype=t.dtype, device=dev)  # a valid pointer for an empty array
        bufs.append(t)
    table = torch.tensor([[b.data_ptr(), hosts[n].rows, hosts[n].cols] for n, b in zip(names, bufs)] or [[0, 0, 0]],
                         dtype=torch.int64).to(dev)
    err = torch.zeros(4, dtype=torch.int64, device=dev)
    width = max(len(r) for r in rows) if rows else 1
    frame_t = torch.tensor([r + [0] * (width - len(r)) for r in rows] or [[0]], dtype=torch.int64).to(dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    launches = 0
    with torch.cuda.device(dev):
        for k, pl in enumerate(plans):
            if pl is None:
                continue
            grid, block = pl
            _lib.jit_launch(h, grid, block, [frame_t[k].data_ptr(), table.data_ptr(), err.data_ptr()],
                            [1, 1, 1], 0, stream)
            launches += 1
        # downloads of the written arrays into one recycled pinned buffer
        sizes = []
        for n, b in zip(names, bufs):
            hh = hosts[n]
            count = hh.rows * (hh.cols if hh.rank == 2 else 1)
            sizes.append(count * b.element_size() * (2 if mode == "dyn" else 1) if n in written else 0)
        pin = _pinned_buffer(sum(sizes) + 64)
        off, views = 0, {}
        for n, b, nb in zip(names, bufs, sizes):
            if nb:
                dst = pin[off:off + nb].view(b.dtype)
                dst.copy_(b.view(-1)[:dst.numel()], non_blocking=True)
                views[n] = dst
                off += (nb + 63) // 64 * 64
        torch.cuda.synchronize(dev)
    e = err.cpu().tolist()
    code = e[0] & 0xFFFFFFFF
    out = {}
    if not code:
        for n in names:
            hh = hosts[n]
            if n not in written:
                out[n] = _host_copy(hh, container)
                continue
            w = views[n].numpy() if n in views else np.zeros(0, dtype=np.int32 if mode == "int32" else np.int64)
            words = w.reshape(-1, 2) if mode == "dyn" else w
            out[n] = _decode(hh, words, mode, pool, container if hh.kind == "zeros" else hh.kind)
    return out, code, e, src, launches, pool


def _dims(loops, env, cap, limit_total):
    """Launch extents for the roles' loops (inner loop on x): the host value of
    each bound where it depends on the environment only, else a default."""
    vals = []
    for _, b, _ in loops:
        try:
            v = host_eval(b, env) if not _has_index(b) else 256
        except (KeyError, ZeroDivisionError):
            v = 256  # depends on an outer meta variable (evaluated in the kernel)
        vals.append(max(1, min(int(v), cap)))
    if not vals:
        return [1]
    if len(vals) == 1:
        return [min(vals[0], limit_total or cap)] if limit_total else [vals[0]]
    inner, outer = vals[1], vals[0]
    if limit_total:
        inner = min(inner, limit_total)
        outer = max(1, min(outer, limit_total // inner))
    return [inner, outer]
