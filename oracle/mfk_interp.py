"""TEST INFRASTRUCTURE ONLY -- a pure-Python restatement of the reference
interpreter for ANY parsed program (the generic path's checker).

Restates parakern.interp (/root/reference/pkg/src/parakern/interp.py) over
the tuple AST of paper_1801_04348_b200.mfk:

* ``c_div`` / ``c_mod``                      interp.py:43-50
* declarations, copies, zero-filled arrays   interp.py:59-81  (Machine.__init__)
* expressions                                interp.py:85-106 (Machine.eval)
* conditions                                 interp.py:108-123 (Machine.test)
* statements, serial loops                   interp.py:129-152 (run_stmt)
* the meta_for nest, lexicographic           interp.py:154-175 (run_schedule, _iterate)
* bounds checks -> IndexError                interp.py:178-212 (_zeros, _deep_copy, _fetch, _put, _checked)

Python's own ints and floats give the reference's value semantics.  Only
tests/ may use this module (it runs small instances: pure-Python loops).
Pinned against the reference's own outputs: tests/golden/generic_vectors.json
(tests/golden/make_generic.py), checked by tests/test_generic.py.
"""

from __future__ import annotations


def c_div(a, b):
    q = abs(a) // abs(b)
    return q if (a >= 0) == (b >= 0) else -q


def c_mod(a, b):
    return a - b * c_div(a, b)


def _zeros(dims):
    if len(dims) == 1:
        return [0] * dims[0]
    return [[0] * dims[1] for _ in range(dims[0])]


def _copy(data):
    data = list(data)
    if data and isinstance(data[0], list):
        return [row[:] for row in data]
    return data[:]


def _checked(i, n, name):
    if not 0 <= i < n:
        raise IndexError("access %s[%d] out of bounds (size %d)" % (name, i, n))
    return i


_I64 = (-(2**63), 2**63 - 1)


class _Machine:
    def __init__(self, prog, params, arrays):
        self.wide = False  # an int result left int64 somewhere (the GPU path raises OverflowError there)
        self.collect = None
        self.env = dict(params)
        self.arrays = {}
        dims = {}
        for kind, name in prog.decl_order:
            if kind == "binding":
                self.env[name] = self.eval(dict(prog.bindings)[name])
            elif kind == "array":
                dims[name] = tuple(self.eval(d) for d in prog.arrays[name])
            elif name not in self.env:
                raise KeyError("no value supplied for parameter %r" % name)
        for name, data in (arrays or {}).items():
            self.arrays[name] = _copy(data)
        for name, d in dims.items():
            if name not in self.arrays:
                self.arrays[name] = _zeros(d)

    def eval(self, e):
        k = e[0]
        if k == "num":
            return e[1]
        if k == "name":
            return self.env[e[1]]
        if k == "bin":
            a, b = self.eval(e[2]), self.eval(e[3])
            op = e[1]
            if op == "+":
                r = a + b
            elif op == "-":
                r = a - b
            elif op == "*":
                r = a * b
            elif op == "/":
                r = c_div(a, b)
            else:
                q = c_div(a, b)
                self._note(b * q)
                r = a - b * q
            self._note(r)
            return r
        idx = tuple(self.eval(s) for s in e[2])
        arr = self.arrays[e[1]]
        try:
            if len(idx) == 1:
                return arr[_checked(idx[0], len(arr), e[1])]
            return arr[_checked(idx[0], len(arr), e[1])][_checked(idx[1], len(arr[0]), e[1])]
        except IndexError:
            raise IndexError("access %s%r out of bounds" % (e[1], idx))

    def _note(self, r):
        if type(r) is int and not _I64[0] <= r <= _I64[1]:
            self.wide = True

    def test(self, c):
        if c[0] == "cmp":
            a, b = self.eval(c[2]), self.eval(c[3])
            return {"<": a < b, "<=": a <= b, ">": a > b, ">=": a >= b, "==": a == b, "!=": a != b}[c[1]]
        return all(self.test(p) for p in c[1])

    def stmts(self, ss):
        for s in ss:
            k = s[0]
            if k == "local":
                self.env[s[1]] = self.eval(s[2])
            elif k == "assign":
                v = self.eval(s[2])
                t = s[1]
                if t[0] == "name":
                    self.env[t[1]] = v
                else:
                    idx = tuple(self.eval(x) for x in t[2])
                    arr = self.arrays[t[1]]
                    if len(idx) == 1:
                        arr[_checked(idx[0], len(arr), t[1])] = v
                    else:
                        arr[_checked(idx[0], len(arr), t[1])][_checked(idx[1], len(arr[0]), t[1])] = v
            elif k == "if":
                if self.test(s[1]):
                    self.stmts(s[2])
                elif s[3] is not None:
                    self.stmts(s[3])
            else:
                for v in range(self.eval(s[2])):
                    self.env[s[1]] = v
                    self.stmts(s[3])

    def nest(self, meta, body):
        if not meta:
            if self.collect is None:
                self.stmts(body)
                return
            # every iteration on its own, errors noted and the walk continued:
            # the exceptions some parallel schedule of this pass can raise
            try:
                self.stmts(body)
            except (IndexError, ZeroDivisionError, KeyError, TypeError) as exc:
                self.collect.add(type(exc))
            return
        var, bound, _ = meta[0]
        for v in range(self.eval(bound)):
            self.env[var] = v
            self.nest(meta[1:], body)

    def context(self, prog, k):
        if k == len(prog.context):
            self.nest(prog.meta, prog.body)
            return
        var, bound = prog.context[k]
        for v in range(self.eval(bound)):
            self.env[var] = v
            self.context(prog, k + 1)


def run_program(prog, params, arrays=None, stats=None, all_iterations=False):
    """interp.run_program for a parsed mfk.Program: the final array contents.
    ``stats`` (a dict) receives ``wide``: whether any int result left int64.
    ``all_iterations``: run every meta_for iteration even after one raised
    (never raising), and put the set of exception types in ``stats["errors"]``."""
    m = _Machine(prog, params, arrays)
    if all_iterations:
        m.collect = set()
        if stats is not None:
            stats["errors"] = m.collect
    try:
        m.context(prog, 0)
    finally:
        if stats is not None:
            stats["wide"] = m.wide
    return m.arrays


def run_block(prog, params, grid_values, context_values=None, arrays=None):
    """interp.run_block (interp.py:228-249): declarations, then the context and
    grid values set, then the thread loops swept over the body."""
    m = _Machine(prog, params, arrays)
    m.env.update(context_values or {})
    m.env.update(grid_values)
    m.nest(list(prog.thread), prog.body)
    return m.arrays
