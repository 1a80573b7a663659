"""Random .mfk programs outside the seven families, and their inputs (test
infrastructure for the generic path: tests/golden/make_generic.py and the
GPU fuzz tests).

Every generated program is race-free in the language's sense (interp.py:12-15):
an iteration of the meta_for nest writes only its own element of the output
(a linear index of the nest variables) and reads arrays no iteration writes in
the same pass, or its own output element -- so the sequential interpreter and
a parallel schedule give the same arrays.  Shapes: 1-D maps over a (grid,
thread) nest, 2-D maps over a 4-deep nest, ping-pong stencils under a serial
context loop (the source half chosen by t % 2), a non-rectangular
(triangular) nest, @grid/@thread annotations, serial loops, if/else and
locals in the body.
"""

from __future__ import annotations

import random

OPS = ["+", "-", "*", "/", "%"]
CMPS = ["<", "<=", ">", ">=", "==", "!="]


class _Gen:
    def __init__(self, rng: random.Random, reads: list, index_vars: list, safe_div: bool, oob: bool):
        self.rng, self.reads, self.vars, self.safe_div, self.oob = rng, reads, index_vars, safe_div, oob
        self.locals: list[str] = []

    def read(self, depth: int) -> str:
        name, size, index_of = self.rng.choice(self.reads)
        r = self.rng.random()
        if self.oob and r < 0.05:
            return "%s[%s]" % (name, index_of(size + self.rng.randint(0, 3)))
        return "%s[%s]" % (name, index_of(None))

    def expr(self, depth: int) -> str:
        r = self.rng.random()
        if depth <= 0 or r < 0.25:
            c = self.rng.random()
            if c < 0.35:
                return self.read(depth)
            if c < 0.55 and self.locals:
                return self.rng.choice(self.locals)
            if c < 0.75:
                return self.rng.choice(self.vars)
            v = self.rng.randint(-9, 9)
            return str(v) if v >= 0 else "(%d)" % v
        op = self.rng.choice(OPS)
        left = self.expr(depth - 1)
        if op in "/%" and self.safe_div:
            right = self.rng.choice(["%d" % self.rng.randint(1, 7), "(%d)" % -self.rng.randint(1, 7),
                                     "(%s * %s + 1)" % ((self.rng.choice(self.vars),) * 2)])
        else:
            right = self.expr(depth - 1)
        return "(%s %s %s)" % (left, op, right)

    def cond(self) -> str:
        parts = ["%s %s %s" % (self.expr(1), self.rng.choice(CMPS), self.expr(1))
                 for _ in range(self.rng.choice([1, 1, 2]))]
        return " && ".join(parts)

    def stmts(self, n: int, depth: int, indent: str) -> list[str]:
        out = []
        for _ in range(n):
            r = self.rng.random()
            if r < 0.45 or depth <= 0:
                name = "x%d" % len(self.locals)
                out.append("%sint %s = %s;" % (indent, name, self.expr(2)))
                self.locals.append(name)
            elif r < 0.6 and self.locals:
                out.append("%s%s = %s;" % (indent, self.rng.choice(self.locals), self.expr(2)))
            elif r < 0.8 and self.locals:
                target = self.rng.choice(self.locals)
                out.append("%sif (%s) {" % (indent, self.cond()))
                out.append("%s    %s = %s;" % (indent, target, self.expr(2)))
                if self.rng.random() < 0.5:
                    out.append("%s} else {" % indent)
                    out.append("%s    %s = %s;" % (indent, target, self.expr(1)))
                out.append("%s}" % indent)
            elif self.locals:
                target = self.rng.choice(self.locals)
                k = "k%d" % self.rng.randint(0, 99)
                self.vars.append(k)
                out.append("%sfor (int %s = 0; %s < %d; %s++)" % (indent, k, k, self.rng.randint(0, 4), k))
                out.append("%s    %s = %s;" % (indent, target, self.expr(1)))
                self.vars.remove(k)
        return out


def program(rng: random.Random, shape: str, safe_div: bool = True, oob: bool = False) -> tuple[str, dict]:
    """(text, params) of one random program of the given shape."""
    if shape == "map1d":
        B = rng.choice([1, 2, 4, 8, 32])
        N = B * rng.randint(1, 24) + rng.choice([0, 0, 3])
        params = {"N": N, "B": B}
        reads = [("a", N, None), ("b", N, None)]
        g = _gen(rng, reads, ["p", "i", "j", "N"], safe_div, oob, N)
        body = ["int p = i * B + j;"] + g.stmts(rng.randint(0, 4), 2, "")
        body.append("c[p] = %s;" % g.expr(3))
        text = ("int N, B;\nint a[N];\nint b[N];\nint c[N];\nint dim = N / B;\n"
                "meta_schedule%s {\n    meta_for (int i = 0; i < dim; i++)\n        meta_for (int j = 0; j < B; j++) {\n"
                % (rng.choice(["", " cache(a)", " cache(a, b)"]))
                + "".join("            %s\n" % l for l in body) + "        }\n}\n")
        return text, params
    if shape == "map2d":
        B0, B1 = rng.choice([1, 2, 4]), rng.choice([1, 2, 8])
        R, C = B0 * rng.randint(1, 6), B1 * rng.randint(1, 6)
        params = {"R": R, "C": C, "B0": B0, "B1": B1}
        g = _Gen(rng, [], ["p", "q", "R", "C"], safe_div, oob)
        g.reads = [("a", R, lambda extra, g=g: "%s][%s" % _two(rng, g, R, C, extra)),
                   ("b", R, lambda extra, g=g: "%s][%s" % _two(rng, g, R, C, extra))]
        body = ["int p = v0 * B0 + u0;", "int q = v1 * B1 + u1;"] + g.stmts(rng.randint(0, 3), 2, "")
        body.append("c[p][q] = %s;" % g.expr(3))
        ann = rng.random() < 0.3
        text = ("int R, C, B0, B1;\nint a[R][C];\nint b[R][C];\nint c[R][C];\nint d0 = R / B0;\nint d1 = C / B1;\n"
                "meta_schedule {\n"
                "    %smeta_for (int v0 = 0; v0 < d0; v0++)\n    %smeta_for (int v1 = 0; v1 < d1; v1++)\n"
                "    %smeta_for (int u0 = 0; u0 < B0; u0++)\n    %smeta_for (int u1 = 0; u1 < B1; u1++) {\n"
                % (("@grid ", "@grid ", "@thread ", "@thread ") if ann else ("", "", "", ""))
                + "".join("        %s\n" % l for l in body) + "    }\n}\n")
        return text, params
    if shape == "stencil":
        B = rng.choice([1, 4, 16])
        N = B * rng.randint(1, 16) + rng.choice([0, 1])
        T = rng.randint(1, 5)
        params = {"N": N, "B": B, "T": T}
        g = _Gen(rng, [], ["p", "t", "N"], safe_div, oob)
        g.reads = [("a", N, lambda extra: "src + %s" % _idx1(rng, "p", N, extra))]
        body = ["int p = i * B + j;", "int src = (t % 2) * N;", "int dst = N - src;"] + g.stmts(rng.randint(0, 3), 2, "")
        body.append("a[dst + p] = %s;" % g.expr(3))
        text = ("int N, B, T;\nint a[2 * N];\nint dim = N / B;\n"
                "for (int t = 0; t < T; t++)\n    meta_schedule cache(a) {\n"
                "        meta_for (int i = 0; i < dim; i++)\n            meta_for (int j = 0; j < B; j++) {\n"
                + "".join("                %s\n" % l for l in body) + "            }\n    }\n")
        return text, params
    if shape == "triangle":
        N = rng.randint(1, 20)
        params = {"N": N}
        g = _gen(rng, [("a", N, None)], ["i", "j", "N"], safe_div, oob, N)
        body = g.stmts(rng.randint(0, 3), 2, "")
        body.append("c[i * N + j] = %s;" % g.expr(3))
        text = ("int N;\nint a[N];\nint c[N * N];\nmeta_schedule {\n    meta_for (int i = 0; i < N; i++)\n"
                "        meta_for (int j = 0; j < i + 1; j++) {\n"
                + "".join("            %s\n" % l for l in body) + "        }\n}\n")
        return text, params
    raise ValueError(shape)


def _idx1(rng, var, n, extra):
    if extra is not None:
        return str(extra)
    return rng.choice(["%s" % var, "(%s + %d) %% %d" % (var, rng.randint(1, 5), n) if n else var,
                       "%d - 1 - %s" % (n, var), "%s / 2" % var, "(%s * 3) %% %d" % (var, n) if n else var])


def _gen(rng, reads, vars_, safe_div, oob, n):
    g = _Gen(rng, [], list(vars_), safe_div, oob)
    g.reads = [(name, size, (lambda extra, size=size: _idx1(rng, "p" if "p" in vars_ else "i", size, extra)))
               for name, size, _ in reads]
    return g


def _two(rng, g, R, C, extra):
    if extra is not None:
        return str(extra), "q"
    return (rng.choice(["p", "(p + 1) %% %d" % R, "%d - 1 - p" % R]),
            rng.choice(["q", "(q + %d) %% %d" % (rng.randint(1, 3), C), "%d - 1 - q" % C]))


def inputs(rng: random.Random, text_params: tuple, style: str) -> dict:
    """Arrays for a generated program: ints (small / wide), floats (with
    specials), mixed int / float lists; declared shapes."""
    text, params = text_params
    shapes = {}
    if "int a[N];" in text:
        shapes["a"] = (params["N"],)
    if "int b[N];" in text:
        shapes["b"] = (params["N"],)
    if "int a[2 * N];" in text:
        shapes["a"] = (2 * params["N"],)
    if "int a[R][C];" in text:
        shapes["a"] = shapes["b"] = (params["R"], params["C"])

    def val():
        if style == "int":
            return rng.randint(-50, 50)
        if style == "wide":
            return rng.choice([rng.randint(-2**40, 2**40), rng.randint(-9, 9)])
        if style == "float":
            return rng.choice([rng.uniform(-10, 10), float(rng.randint(-5, 5)), 0.5, -0.0, 1e300])
        return rng.choice([rng.randint(-20, 20), rng.uniform(-5, 5)])

    out = {}
    for name, shp in shapes.items():
        if len(shp) == 1:
            out[name] = [val() for _ in range(shp[0])]
        else:
            out[name] = [[val() for _ in range(shp[1])] for _ in range(shp[0])]
    return out
