"""Front end for ``.mfk`` programs, self-contained (no parakern at run time).

The language is the reference's annotated loop-nest fragment
(/root/reference/pkg/src/parakern/dsl.py:1-30): integer declarations, derived
bindings, serial context loops around exactly one ``meta_schedule``, a
perfect nest of 1-4 ``meta_for`` loops with canonical headers, and a body of
locals, assignments, ``if``/``else`` and serial ``for`` loops.  This module
parses it into a small tuple AST and applies the checks the reference's
``dsl.parse`` applies (``_Parser``, dsl.py:275-598; ``_validate_nest``,
dsl.py:605-629; ``split_roles``, dsl.py:632-657), so a text is accepted
exactly when the reference accepts it (pinned: tests/golden/parse_vectors.json).

It feeds ``generic.py``, the GPU path for programs outside the seven
hand-written kernel families.  Classification rules that only the reference's
optimizer applies (``classify_parameters``: read-only parameters, data vs
program split) are not parse errors there and are not applied here either:
``interp.run_program`` executes any parsed program.

AST (tuples, first field the node kind):

  expr  ('num', v) | ('name', id) | ('bin', op, l, r) | ('idx', array, (subs...))
  cond  ('cmp', op, l, r) | ('and', (cmp, ...))
  stmt  ('local', name, e) | ('assign', target, e) | ('if', cond, then, orelse | None)
        | ('for', var, bound, stmts)
"""

from __future__ import annotations

import re
from dataclasses import dataclass, field

__all__ = ["MfkError", "Program", "parse"]

KEYWORDS = frozenset({"int", "for", "if", "else", "meta_schedule", "meta_for", "cache"})

_LEX = re.compile(r"(?P<nl>\n)|(?P<ws>[ \t\r]+)|(?P<cm>//[^\n]*)|(?P<num>\d+)|(?P<id>[A-Za-z_]\w*)"
                  r"|(?P<op>\+\+|&&|<=|>=|==|!=|[-+*/%<>=;,(){}\[\]@])")


class MfkError(ValueError):
    """A program the language does not accept (the reference's DslError)."""

    def __init__(self, message: str, line: int | None = None, col: int | None = None):
        super().__init__(message if line is None else "line %d, col %d: %s" % (line, col, message))
        self.line, self.col = line, col


def _tokens(text: str) -> list:
    """(kind, text, line, col) with kind num | id | kw | op | eof."""
    out, line, col, pos = [], 1, 1, 0
    while pos < len(text):
        m = _LEX.match(text, pos)
        if m is None:
            raise MfkError("unexpected character %r" % text[pos], line, col)
        kind, tok = m.lastgroup, m.group(0)
        if kind == "nl":
            line, col = line + 1, 1
        else:
            if kind not in ("ws", "cm"):
                out.append(("kw" if kind == "id" and tok in KEYWORDS else kind, tok, line, col))
            col += len(tok)
        pos = m.end()
    out.append(("eof", "", line, col))
    return out


@dataclass
class Program:
    """A parsed program, with the pieces the executor needs."""

    scalars: list                    # declared scalar names, declaration order
    arrays: dict                     # name -> (dim expr, ...) (1 or 2 dims), declaration order
    bindings: list                   # [(name, expr)] in order
    context: list                    # [(var, bound)] serial loops enclosing the schedule, outermost first
    cache: tuple                     # names in cache(...) (a staging hint; no effect on results)
    meta: list                       # [(var, bound, role)] the meta_for nest, outermost first
    body: tuple                      # statements of the innermost meta_for
    grid: list = field(default_factory=list)    # meta entries on the grid (<= 2)
    thread: list = field(default_factory=list)  # meta entries on the thread block (<= 2)
    decl_order: list = field(default_factory=list)  # ('scalar'|'array'|'binding', name) as written


class _Parser:
    def __init__(self, text: str):
        self.t = _tokens(text)
        self.i = 0

    # -- plumbing --
    def peek(self, k: int = 0):
        return self.t[min(self.i + k, len(self.t) - 1)]

    def at(self, kind: str, text: str | None = None) -> bool:
        tk = self.peek()
        return tk[0] == kind and (text is None or tk[1] == text)

    def take(self):
        tk = self.t[self.i]
        if tk[0] != "eof":
            self.i += 1
        return tk

    def want(self, kind: str, text: str | None = None):
        if not self.at(kind, text):
            tk = self.peek()
            raise MfkError("expected %r, found %r" % (text if text is not None else kind, tk[1] or "<eof>"),
                           tk[2], tk[3])
        return self.take()

    def err(self, msg: str, tk=None) -> MfkError:
        tk = tk or self.peek()
        return MfkError(msg, tk[2], tk[3])

    # -- declarations and the top level --
    def program(self) -> Program:
        scalars, arrays, bindings, order = [], {}, [], []
        while self.at("kw", "int"):
            self.take()
            while True:
                name = self.want("id")[1]
                if self.at("op", "["):
                    dims = [self.bracket()]
                    if self.at("op", "["):
                        dims.append(self.bracket())
                    arrays[name] = tuple(dims)
                    order.append(("array", name))
                elif self.at("op", "="):
                    self.take()
                    bindings.append((name, self.expr()))
                    order.append(("binding", name))
                else:
                    scalars.append(name)
                    order.append(("scalar", name))
                if self.at("op", ","):
                    self.take()
                    continue
                self.want("op", ";")
                break
        found = []  # (context loops, schedule)
        while not self.at("eof"):
            self.top_statement([], found)
        if len(found) != 1:
            raise MfkError("program must contain exactly one meta_schedule (found %d)" % len(found))
        context, (cache, meta, body) = found[0]
        prog = Program(scalars, arrays, bindings, context, cache, meta, body, decl_order=order)
        _check_nest(prog)
        return prog

    def bracket(self):
        self.want("op", "[")
        e = self.expr()
        self.want("op", "]")
        return e

    def top_statement(self, context: list, found: list) -> None:
        if self.at("kw", "for"):
            self.take()
            var, bound = self.header()
            inner = context + [(var, bound)]
            if self.at("op", "{"):
                self.take()
                while not self.at("op", "}"):
                    self.top_statement(inner, found)
                self.take()
            else:
                self.top_statement(inner, found)
            return
        if self.at("kw", "meta_schedule"):
            found.append((list(context), self.schedule()))
            return
        raise self.err("expected a serial 'for' or 'meta_schedule' at the top level")

    def header(self):
        """``(int v = 0; v < bound; v++)`` or ``++v``."""
        self.want("op", "(")
        self.want("kw", "int")
        var = self.want("id")[1]
        self.want("op", "=")
        z = self.peek()
        if not (z[0] == "num" and z[1] == "0"):
            raise self.err("loops must start at 0", z)
        self.take()
        self.want("op", ";")
        c = self.want("id")
        if c[1] != var:
            raise self.err("loop condition must test %r" % var, c)
        self.want("op", "<")
        bound = self.expr()
        self.want("op", ";")
        if self.at("op", "++"):
            self.take()
            s = self.want("id")
        else:
            s = self.want("id")
            self.want("op", "++")
        if s[1] != var:
            raise self.err("loop increment must step %r" % var, s)
        self.want("op", ")")
        return var, bound

    def schedule(self):
        self.want("kw", "meta_schedule")
        cache = ()
        if self.at("kw", "cache"):
            self.take()
            self.want("op", "(")
            names = [self.want("id")[1]]
            while self.at("op", ","):
                self.take()
                names.append(self.want("id")[1])
            self.want("op", ")")
            cache = tuple(names)
        self.want("op", "{")
        if not (self.at("kw", "meta_for") or self.at("op", "@")):
            raise self.err("meta_schedule body must begin with meta_for")
        meta = []
        body = self.meta_for(meta)
        self.want("op", "}")
        return cache, meta, body

    def meta_for(self, meta: list) -> tuple:
        role = None
        if self.at("op", "@"):
            at = self.take()
            ann = self.want("id")
            if ann[1] not in ("grid", "thread"):
                raise self.err("unknown annotation @%s (use @grid or @thread)" % ann[1], at)
            role = ann[1]
        self.want("kw", "meta_for")
        var, bound = self.header()
        meta.append((var, bound, role))
        if self.at("kw", "meta_for") or self.at("op", "@"):
            return self.meta_for(meta)
        if self.at("op", "{"):
            self.take()
            if self.at("kw", "meta_for") or self.at("op", "@"):
                body = self.meta_for(meta)
                if not self.at("op", "}"):
                    raise self.err("meta_for nest must be a perfect prefix of the loop tree")
                self.take()
                return body
            stmts = []
            while not self.at("op", "}"):
                stmts.append(self.statement())
            self.take()
            return tuple(stmts)
        return (self.statement(),)

    # -- body statements --
    def block(self) -> tuple:
        if self.at("op", "{"):
            self.take()
            stmts = []
            while not self.at("op", "}"):
                stmts.append(self.statement())
            self.take()
            return tuple(stmts)
        return (self.statement(),)

    def statement(self) -> tuple:
        if self.at("kw", "meta_for") or self.at("kw", "meta_schedule"):
            raise self.err("%s not allowed inside a loop body" % self.peek()[1])
        if self.at("kw", "int"):
            self.take()
            name = self.want("id")[1]
            self.want("op", "=")
            e = self.expr()
            self.want("op", ";")
            return ("local", name, e)
        if self.at("kw", "for"):
            self.take()
            var, bound = self.header()
            return ("for", var, bound, self.block())
        if self.at("kw", "if"):
            self.take()
            self.want("op", "(")
            cond = self.condition()
            self.want("op", ")")
            then = self.block()
            orelse = None
            if self.at("kw", "else"):
                self.take()
                orelse = self.block()
            return ("if", cond, then, orelse)
        name = self.want("id")[1]
        target = ("idx", name, self.subscripts()) if self.at("op", "[") else ("name", name)
        self.want("op", "=")
        e = self.expr()
        self.want("op", ";")
        return ("assign", target, e)

    def subscripts(self) -> tuple:
        subs = [self.bracket()]
        if self.at("op", "["):
            subs.append(self.bracket())
        return tuple(subs)

    def condition(self):
        parts = [self.comparison()]
        while self.at("op", "&&"):
            self.take()
            parts.append(self.comparison())
        return parts[0] if len(parts) == 1 else ("and", tuple(parts))

    def comparison(self):
        left = self.expr()
        tk = self.peek()
        if tk[0] == "op" and tk[1] in ("<", "<=", ">", ">=", "==", "!="):
            self.take()
            return ("cmp", tk[1], left, self.expr())
        raise self.err("expected a comparison operator", tk)

    def expr(self):
        e = self.term()
        while self.at("op", "+") or self.at("op", "-"):
            op = self.take()[1]
            e = ("bin", op, e, self.term())
        return e

    def term(self):
        e = self.unary()
        while self.at("op", "*") or self.at("op", "/") or self.at("op", "%"):
            op = self.take()[1]
            e = ("bin", op, e, self.unary())
        return e

    def unary(self):
        if self.at("op", "-"):
            self.take()
            inner = self.unary()
            # a negated literal folds into the literal (dsl.py:576-581)
            return ("num", -inner[1]) if inner[0] == "num" else ("bin", "-", ("num", 0), inner)
        return self.atom()

    def atom(self):
        tk = self.peek()
        if tk[0] == "num":
            self.take()
            return ("num", int(tk[1]))
        if tk[0] == "id":
            self.take()
            return ("idx", tk[1], self.subscripts()) if self.at("op", "[") else ("name", tk[1])
        if self.at("op", "("):
            self.take()
            e = self.expr()
            self.want("op", ")")
            return e
        raise self.err("expected an expression", tk)


def _check_nest(prog: Program) -> None:
    """The nest checks of dsl.parse (dsl.py:605-629): depth 1-4, all-or-none
    annotations with @grid outside @thread, distinct variables; the roles as
    dsl.split_roles assigns them (dsl.py:632-657: as annotated, else the outer
    half of the nest, rounded up, on the grid)."""
    meta = prog.meta
    if not 1 <= len(meta) <= 4:
        raise MfkError("meta_for nest depth must be between 1 and 4 (got %d)" % len(meta))
    roles = [r for _, _, r in meta]
    if any(r is not None for r in roles):
        if any(r is None for r in roles):
            raise MfkError("either annotate every meta_for with @grid/@thread or none")
        inside = False
        for r in roles:
            if r == "thread":
                inside = True
            elif inside:
                raise MfkError("@grid meta_for cannot appear inside @thread")
        if roles[0] != "grid":
            raise MfkError("the outermost meta_for must be @grid")
    seen = set()
    for var, _, _ in meta:
        if var in seen:
            raise MfkError("duplicate meta_for variable %r" % var)
        seen.add(var)
    if roles[0] is not None:
        grid = [m for m in meta if m[2] == "grid"]
        thread = [m for m in meta if m[2] == "thread"]
    else:
        k = (len(meta) + 1) // 2
        grid, thread = list(meta[:k]), list(meta[k:])
    # more than two of a role is legal text (dsl.split_roles refuses it only
    # when the optimizer maps the nest; interp.run_program runs it): the
    # executor runs the extra loops serially inside each thread
    prog.grid, prog.thread = grid, thread


def parse(text: str) -> Program:
    """Parse ``.mfk`` text; ``MfkError`` where the reference's dsl.parse raises DslError."""
    return _Parser(text).program()


# ------------------------------------------------------------------ walks ---

def walk_exprs(node):
    """Every expression node under an expr / cond / stmt / statement tuple."""
    if isinstance(node, tuple) and node and isinstance(node[0], str):
        k = node[0]
        if k in ("num", "name"):
            yield node
        elif k == "bin":
            yield node
            yield from walk_exprs(node[2])
            yield from walk_exprs(node[3])
        elif k == "idx":
            yield node
            for s in node[2]:
                yield from walk_exprs(s)
        elif k == "cmp":
            yield from walk_exprs(node[2])
            yield from walk_exprs(node[3])
        elif k == "and":
            for p in node[1]:
                yield from walk_exprs(p)
        elif k == "local":
            yield from walk_exprs(node[2])
        elif k == "assign":
            yield from walk_exprs(node[1])
            yield from walk_exprs(node[2])
        elif k == "if":
            yield from walk_exprs(node[1])
            for s in node[2]:
                yield from walk_exprs(s)
            for s in node[3] or ():
                yield from walk_exprs(s)
        elif k == "for":
            yield from walk_exprs(node[2])
            for s in node[3]:
                yield from walk_exprs(s)
    elif isinstance(node, tuple):
        for s in node:
            yield from walk_exprs(s)


def render_expr(e) -> str:
    """C text of an expression (fully parenthesised)."""
    k = e[0]
    if k == "num":
        return str(e[1])
    if k == "name":
        return e[1]
    if k == "bin":
        return "(%s %s %s)" % (render_expr(e[2]), e[1], render_expr(e[3]))
    return e[1] + "".join("[%s]" % render_expr(s) for s in e[2])
