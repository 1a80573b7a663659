"""GPU path for programs outside the seven hand-written families.

SURVEY 8(f) row 2.  The reference renders a case's program as CUDA-C
(``parakern.emit.emit_kernel``, pkg/src/parakern/emit.py:268-363) but never
compiles it.  Here that text is compiled for sm_100a at load time with NVRTC
(``pk_jit_compile``) and launched with the emitter's own geometry
(``_launch_stanza``, emit.py:561-594): grid = the grid meta_for bounds capped
at PK_GRID_STRIDE, block = the thread meta_for bounds, one launch per
iteration of the serial context loops.  The same machinery runs the
emitted kernels of the seven families as the "naive emitted kernel"
baseline the hand-written kernels are measured against.

Leaf choice.  The emitter stages cached arrays in STATIC shared memory, so
the case discussion is evaluated with Z_B = 48 KB / 4 (the static limit).
Only leaves that keep the program's own parameters are used here -- the
original program, or the same program with caching-off -- because a
granularity leaf needs a program-specific parameter remap (e.g. B' = s*B,
pkg/tests/test_acceptance.py:400-408) to preserve results in general.

A ``Leaf`` is self-contained (source text + launch description), so leaves
can be generated where parakern is installed and run anywhere.
"""

from __future__ import annotations

import re
from dataclasses import asdict, dataclass, field

from . import _lib

# ---------------------------------------------------------------- C exprs ----

from .programs import c_div  # noqa: E402

_TOK = re.compile(r"\s*(\d+|[A-Za-z_][A-Za-z_0-9]*|[-+*/%()])")


def _c_div(a: int, b: int) -> int:
    if b == 0:
        raise ZeroDivisionError("division by zero in a binding (interp.py:43-46)")
    return c_div(a, b)


def ceval(text: str, env: dict) -> int:
    """Evaluate a DSL expression (dsl.render_expr text) with C semantics."""
    toks = [m.group(1) for m in _TOK.finditer(text)]
    pos = 0

    def peek():
        return toks[pos] if pos < len(toks) else None

    def take():
        nonlocal pos
        pos += 1
        return toks[pos - 1]

    def factor():
        t = take()
        if t == "(":
            v = expr()
            take()
            return v
        if t == "-":
            return -factor()
        if t.isdigit():
            return int(t)
        if t not in env:
            raise KeyError("no value supplied for parameter %r" % t)
        return int(env[t])

    def term():
        v = factor()
        while peek() in ("*", "/", "%"):
            op = take()
            r = factor()
            if op == "*":
                v = v * r
            elif op == "/":
                v = _c_div(v, r)
            else:
                v = v - r * _c_div(v, r)
        return v

    def expr():
        v = term()
        while peek() in ("+", "-"):
            op = take()
            r = term()
            v = v + r if op == "+" else v - r
        return v

    return expr()


# ------------------------------------------------------------------- leaf ----

@dataclass
class Leaf:
    """One emitted kernel and how to launch it."""

    kernel_name: str
    source: str                      # preamble + kernel text
    params: list                     # scalar parameters (declaration order)
    arrays: list                     # [(name, [dim expr, ...])]
    bindings: list                   # [(name, expr)]
    grid: list                       # [(var, bound expr)] outermost first
    thread: list                     # [(var, bound expr)] outermost first
    context: list                    # [(var, bound expr)] serial loops around the schedule
    args: list                       # [(name, kind)] kernel formals, kind 'ptr' | 'int'
    macros: list                     # parameters the emitter wants as -DPK_<name>
    grid_stride: int = 256
    applied: list = field(default_factory=list)

    def to_json(self) -> dict:
        return asdict(self)

    @classmethod
    def from_json(cls, d: dict) -> "Leaf":
        return cls(**{k: d[k] for k in cls.__dataclass_fields__ if k in d})


def leaf_from_kernel_text(kt, case_program, name: str, grid_stride: int = 256, applied=()) -> Leaf:
    """Build a Leaf from parakern's KernelText and the case's program (needs parakern)."""
    from parakern import dsl, model

    cfg = model.build_source_cfg(case_program)
    table = dsl.classify_parameters(case_program)
    sig = re.search(r"__global__ void (\w+)\(([^)]*)\)", kt.kernel)
    kname, formals = sig.group(1), sig.group(2)
    args = []
    for f in (x.strip() for x in formals.split(",") if x.strip()):
        if f.startswith("int *"):
            args.append((f[5:].strip(), "ptr"))
        else:
            args.append((f.split()[-1], "int"))
    macros = re.findall(r"#ifndef PK_(\w+)\n#error", kt.preamble)
    kernel = kt.kernel
    # The emitter's formals (_scalar_formals, emit.py) omit parameters used
    # only as a 2-D row pitch (e.g. matmul's n in c[p * n + q]); the text
    # would not compile.  Append every program parameter / binding the body
    # names but the signature lacks.
    declared = {a for a, _ in args}
    body = kernel[kernel.index("{"):]
    scalars = list(table.order) + [b for b, _ in table.bindings]
    extra = [s for s in scalars if s not in declared and re.search(r"\b%s\b" % re.escape(s), body)]
    if extra:
        new_formals = formals + "".join(", int %s" % s for s in extra)
        kernel = kernel.replace("(%s)" % formals, "(%s)" % new_formals, 1)
        args += [(s, "int") for s in extra]
    return Leaf(
        kernel_name=kname,
        source=kt.preamble + "\n" + kernel + "\n",
        params=list(table.order),
        arrays=[(a, [dsl.render_expr(d) for d in dims]) for a, dims in table.arrays.items()],
        bindings=[(b, dsl.render_expr(v)) for b, v in table.bindings],
        grid=[(m.var, dsl.render_expr(m.bound)) for m in cfg.grid],
        thread=[(m.var, dsl.render_expr(m.bound)) for m in cfg.thread],
        context=[(c.var, dsl.render_expr(c.bound)) for c in cfg.context],
        args=args,
        macros=macros,
        grid_stride=grid_stride,
        applied=list(applied),
    )


def emit_leaf(program, params: dict, *, z_words: int = 12288, name: str = "pk_jit") -> Leaf:
    """Run the reference's engine + emitter for ``program`` (parakern needed):
    the original program if its cached footprint fits ``z_words`` of static
    shared memory, else the same program with caching-off."""
    from fractions import Fraction

    from parakern import counters, dsl, emit, model, strategies
    from parakern.machine import parse_machine

    from . import machine as machine_mod

    mv = machine_mod.MachineValues("b200", {"Z_B": z_words, "R_B": 255, "T_B": 1024}, "static")
    mspec = parse_machine(machine_mod.machine_file_text(mv))
    table = dsl.classify_parameters(program)
    prog, applied = program, ()
    if program.schedule.cache:
        cfg = model.build_source_cfg(program)
        layout = counters.footprint_layout(cfg, table, mspec.box(table.order))
        words = layout.total.eval({k: Fraction(int(params[k])) for k in table.order})
        if words > z_words:
            prog, applied = strategies.apply_source("caching-off", program), ("caching-off",)

    class _Case:  # the attributes emit_kernel reads from an engine.Case
        index = 1

    c = _Case()
    c.program = prog
    c.applied = applied
    kt = emit.emit_kernel(c, mspec, name=name)
    return leaf_from_kernel_text(kt, prog, name, mspec.grid_stride, applied)


# -------------------------------------------------------------------- run ----

_compiled: dict = {}


def compile_leaf(leaf: Leaf, env: dict) -> int:
    opts = ["-DNDEBUG"] + ["-DPK_%s=%d" % (m, int(env[m])) for m in leaf.macros]
    key = (leaf.source, tuple(opts))
    h = _compiled.get(key)
    if h is None:
        # NVRTC has no host headers; the emitted asserts only re-check the -DPK_*
        # macros against the arguments, which run_leaf derives from the same values
        src = leaf.source.replace("#include <assert.h>", "#define assert(x) ((void)0)")
        # unmangled symbol so the module lookup finds the emitter's kernel name
        src = src.replace("__global__ void " + leaf.kernel_name + "(",
                          'extern "C" __global__ void ' + leaf.kernel_name + "(")
        h = _lib.jit_compile(src, leaf.kernel_name, opts)
        _compiled[key] = h
    return h


def run_leaf(leaf: Leaf, params: dict, buffers: dict, stream: int = 0) -> int:
    """Launch an emitted leaf on device buffers (name -> torch int32 tensor).
    Returns the number of kernel launches."""
    env = {p: int(params[p]) for p in leaf.params if p in params}
    missing = [p for p in leaf.params if p not in params]
    if missing:
        raise KeyError("no value supplied for parameter %r" % missing[0])
    for b, expr in leaf.bindings:
        env[b] = ceval(expr, env)
    grid = [max(0, min(ceval(e, env), leaf.grid_stride)) for _, e in leaf.grid]
    block = [max(0, ceval(e, env)) for _, e in leaf.thread]
    if any(g == 0 for g in grid) or any(b == 0 for b in block):
        return 0  # an empty meta_for: nothing runs (interp.py:166-174)
    if block and eval_product(block) > 1024:
        raise ValueError("thread block of %d threads exceeds T_B = 1024" % eval_product(block))
    h = compile_leaf(leaf, env)
    gdim = list(reversed(grid))   # dimGrid(inner, outer), emit.py:585
    bdim = list(reversed(block))  # dimBlock(B1, B0)

    def launch(e):
        vals, kinds = [], []
        for name, kind in leaf.args:
            if kind == "ptr":
                vals.append(buffers[name].data_ptr())
                kinds.append(1)
            else:
                vals.append(e[name])
                kinds.append(0)
        _lib.jit_launch(h, gdim, bdim, vals, kinds, 0, stream)

    count = 0

    def loops(i, e):
        nonlocal count
        if i == len(leaf.context):
            launch(e)
            count += 1
            return
        var, bound = leaf.context[i]
        for v in range(ceval(bound, e)):
            e2 = dict(e)
            e2[var] = v
            loops(i + 1, e2)

    loops(0, env)
    return count


# -------------------------------------------------------------- run_block --

_packaged: dict = {}


def packaged_leaf(family: str, variant: str) -> Leaf:
    """The reference emitter's leaf for a family's original program or its
    caching-off case program (data/leaves.json, tools/export_leaves.py)."""
    import json
    import os

    if not _packaged:
        path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "data", "leaves.json")
        with open(path) as fh:
            _packaged.update(json.load(fh)["leaves"])
    key = "%s/%s" % (family, variant)
    if key not in _packaged:
        raise NotImplementedError("no emitted leaf for %s (%s)" % (family, variant))
    return Leaf.from_json(_packaged[key])


_GRID_LOOP = re.compile(r"for \(int (\w+) = \(int\)blockIdx\.[xyz]; \1 < [^;]+; \1 \+= PK_GRID_STRIDE\)")


def block_leaf(leaf: Leaf) -> Leaf:
    """The same kernel with every grid meta_for pinned to one value (a kernel
    argument pk_rb_<var>): launched as one block it runs exactly the body
    instances interp.run_block sweeps (grid indices fixed, thread loops over
    the block's threads, interp.py:228-249)."""
    vars_ = [v for v, _ in leaf.grid]
    src, n = _GRID_LOOP.subn(lambda m: "for (int {0} = pk_rb_{0}, pk_once_{0} = 1; pk_once_{0}; pk_once_{0} = 0)"
                             .format(m.group(1)), leaf.source)
    if n != len(vars_):
        raise NotImplementedError("emitted grid loops of %s not in the expected form" % leaf.kernel_name)
    sig = re.search(r"(__global__ void %s\()([^)]*)\)" % re.escape(leaf.kernel_name), src)
    src = src[:sig.end(2)] + "".join(", int pk_rb_%s" % v for v in vars_) + src[sig.end(2):]
    b = Leaf(**{k: getattr(leaf, k) for k in Leaf.__dataclass_fields__})
    b.source = src
    b.args = list(leaf.args) + [("pk_rb_%s" % v, "int") for v in vars_]
    return b


def run_block_leaf(leaf: Leaf, params: dict, grid_values: dict, context_values: dict, buffers: dict,
                   stream: int = 0) -> None:
    """One block of an emitted leaf (see block_leaf) on device buffers."""
    env = {p: int(params[p]) for p in leaf.params if p in params}
    missing = [p for p in leaf.params if p not in params]
    if missing:
        raise KeyError("no value supplied for parameter %r" % missing[0])
    for b, expr in leaf.bindings:
        env[b] = ceval(expr, env)
    roles = [(v, b, grid_values) for v, b in leaf.grid] + [(v, b, context_values) for v, b in leaf.context]
    for var, bound, src in roles:
        if var not in src:
            raise KeyError("no value supplied for %r" % var)
        v, hi = int(src[var]), ceval(bound, env)
        # outside its loop's range the reference runs the body anyway and
        # raises IndexError only if an access leaves its array; here such a
        # block is refused before it runs
        if not 0 <= v < hi:
            raise IndexError("%s = %d outside its loop range [0, %d)" % (var, v, hi))
        env[var] = v
    block = [max(0, ceval(e, env)) for _, e in leaf.thread]
    if any(x == 0 for x in block):
        return  # an empty thread meta_for: nothing runs
    if eval_product(block) > 1024:
        raise ValueError("thread block of %d threads exceeds T_B = 1024" % eval_product(block))
    bl = block_leaf(leaf)
    h = compile_leaf(bl, env)
    for var, _ in leaf.grid:
        env["pk_rb_" + var] = env[var]
    vals, kinds = [], []
    for name, kind in bl.args:
        if kind == "ptr":
            vals.append(buffers[name].data_ptr())
            kinds.append(1)
        else:
            vals.append(env[name])
            kinds.append(0)
    _lib.jit_launch(h, [1] * len(leaf.grid), list(reversed(block)), vals, kinds, 0, stream)


def eval_product(xs) -> int:
    p = 1
    for x in xs:
        p *= x
    return p


def array_shapes(leaf: Leaf, params: dict) -> dict:
    env = {p: int(params[p]) for p in leaf.params if p in params}
    for b, expr in leaf.bindings:
        env[b] = ceval(expr, env)
    return {a: tuple(max(0, ceval(d, env)) for d in dims) for a, dims in leaf.arrays}


def run_program_jit(leaf: Leaf, params: dict, arrays: dict | None = None):
    """run_program semantics for an emitted leaf: fresh arrays, zeros for the
    ones not supplied, results as int lists / numpy like the inputs."""
    import numpy as np
    import torch

    from .interp import _to_device_tensor

    arrays = arrays or {}
    shapes = array_shapes(leaf, params)
    bufs = {}
    dev = torch.device("cuda", torch.cuda.current_device())
    for name, shape in shapes.items():
        n = eval_product(shape)
        if name in arrays:
            # the emitted leaves carry no bounds guards: an array shorter than
            # its declaration raises IndexError here (interp.py:209-212) instead
            # of letting the kernel run past the buffer; values outside int32
            # raise OverflowError instead of wrapping
            t, _ = _to_device_tensor(name, arrays[name], shape, np.int32, dev)
            bufs[name] = t[: max(n, 1)].contiguous() if t.numel() > n else t
        else:
            bufs[name] = torch.zeros(max(n, 1), dtype=torch.int32, device="cuda")
    stream = torch.cuda.current_stream().cuda_stream
    run_leaf(leaf, params, bufs, stream)
    torch.cuda.synchronize()
    out = {}
    for name, v in arrays.items():  # arrays the program does not declare come back as copies
        if name not in shapes:
            out[name] = v.copy() if isinstance(v, np.ndarray) else [r[:] if isinstance(r, list) else r for r in v]
    for name, shape in shapes.items():
        host = bufs[name].cpu().numpy()[: eval_product(shape)].reshape(shape)
        out[name] = host.tolist() if not isinstance(arrays.get(name), np.ndarray) else host
    return out
