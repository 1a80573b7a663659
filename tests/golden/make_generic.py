"""Generate tests/golden/generic_vectors.json from the REFERENCE front end and
interpreter: programs outside the seven families (the generic path).

For every program text of a corpus -- hand-written programs covering the
language (annotations, if/else, && chains, serial loops, locals, every
operator on negative operands, triangular nests, context loops), random
race-free programs (tests/generic_programs.py), and texts the language
rejects -- this script records

* ``parakern.dsl.parse`` (dsl.py:601): accepted or rejected (DslError), and
  for accepted texts the structure the executor relies on: scalars,
  arrays, bindings, context loop variables, meta_for variables with their
  grid / thread roles (``dsl.split_roles``, dsl.py:632-657);
* ``parakern.interp.run_program`` (interp.py:215) on seeded inputs of
  several value styles (ints, wide ints, binary64 floats with specials,
  mixed int / float lists, bools and other objects moved): the arrays, or
  the exception it raises.

Only this script touches /root/reference.

    python tests/golden/make_generic.py [--ref /root/reference/pkg/src]
"""

from __future__ import annotations

import argparse
import json
import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(HERE))

import generic_programs  # noqa: E402

HAND = [
    # scale-and-shift with every operator on negative operands, @grid/@thread
    ("ops", """int N, B;
int a[N];
int c[N];
int d = N / B;
meta_schedule {
    @grid meta_for (int i = 0; i < d; i++)
        @thread meta_for (int j = 0; j < B; j++) {
            int p = i * B + j;
            int x = a[p];
            c[p] = (x / 3) * 1000000 + (x % 3) * 10000 + (x / (-3)) * 100 + x % (-3);
        }
}
""", {"N": 24, "B": 4}),
    # if / else with an && chain, a serial loop accumulating into a local
    ("branch", """int N;
int a[N];
int c[N];
meta_schedule {
    meta_for (int i = 0; i < N; i++) {
        int acc = 0;
        for (int k = 0; k < 4; k++)
            acc = acc + a[(i + k) % N] * (k - 1);
        if (acc > 10 && a[i] != 0) {
            c[i] = acc / a[i];
        } else {
            if (acc <= -10)
                c[i] = acc % 7;
            else
                c[i] = acc;
        }
    }
}
""", {"N": 17}),
    # triangular nest (a bound that reads an outer meta variable)
    ("triangle", """int N;
int a[N];
int c[N * N];
meta_schedule {
    meta_for (int i = 0; i < N; i++)
        meta_for (int j = 0; j < i + 1; j++)
            c[i * N + j] = a[i] * a[j] - i * j;
}
""", {"N": 9}),
    # two context loops around a ping-pong 2-D smoothing step
    ("pingpong2d", """int T, R, C;
int a[2 * R][C];
for (int t = 0; t < T; t++)
    for (int u = 0; u < 2; u++)
        meta_schedule {
            meta_for (int r = 0; r < R; r++)
                meta_for (int q = 0; q < C; q++) {
                    int s = ((2 * t + u) % 2) * R;
                    int d = R - s;
                    a[d + r][q] = (a[s + r][q] + a[s + (r + 1) % R][q] + a[s + r][(q + C - 1) % C]) / 3;
                }
        }
""", {"T": 3, "R": 6, "C": 5}),
    # a scalar parameter never read, a binding of bindings, a 3-deep nest
    ("nest3", """int N, M, unused;
int a[N][M];
int c[N][M];
int h = N / 2;
int hh = h + h;
meta_schedule {
    meta_for (int i = 0; i < hh; i++)
        meta_for (int j = 0; j < M; j++)
            meta_for (int k = 0; k < 1; k++)
                c[i][j] = a[hh - 1 - i][j] + k;
}
""", {"N": 7, "M": 3, "unused": 5}),
    # moves only: any object goes through unchanged
    ("move", """int N;
int a[N];
int c[N];
meta_schedule {
    meta_for (int i = 0; i < N; i++)
        c[N - 1 - i] = a[i];
}
""", {"N": 8}),
]

BAD = [
    "int N;\nint a[N];\nmeta_schedule { meta_for (int i = 1; i < N; i++) a[i] = 0; }\n",   # loop from 1
    "int N;\nint a[N];\nmeta_schedule { meta_for (int i = 0; i <= N; i++) a[i] = 0; }\n",  # <= bound
    "int N;\nint a[N];\nfor (int t = 0; t < 2; t++) a[0] = 1;\n",                          # no schedule
    "int N;\nint a[N];\nmeta_schedule { meta_for (int i = 0; i < N; i++) a[i] = 0; }\n"
    "meta_schedule { meta_for (int j = 0; j < N; j++) a[j] = 1; }\n",                      # two schedules
    "int N;\nint a[N];\nmeta_schedule { meta_for (int i = 0; i < N; i++) "
    "meta_for (int j = 0; j < N; j++) meta_for (int k = 0; k < N; k++) meta_for (int l = 0; l < N; l++) "
    "meta_for (int m = 0; m < N; m++) a[i] = 0; }\n",                                       # depth 5
    "int N;\nint a[N];\nmeta_schedule { @grid meta_for (int i = 0; i < N; i++) meta_for (int j = 0; j < N; j++) "
    "a[i] = j; }\n",                                                                          # partial annotation
    "int N;\nint a[N];\nmeta_schedule { @thread meta_for (int i = 0; i < N; i++) @grid meta_for (int j = 0; j < N; "
    "j++) a[i] = j; }\n",                                                                     # grid inside thread
    "int N;\nint a[N];\nmeta_schedule { meta_for (int i = 0; i < N; i++) meta_for (int i = 0; i < N; i++) "
    "a[i] = 0; }\n",                                                                          # duplicate variable
    "int N;\nint a[N];\nmeta_schedule { meta_for (int i = 0; i < N; i++) { int x = 1; meta_for (int j = 0; "
    "j < N; j++) a[i] = x; } }\n",                                                            # imperfect nest
    "int N;\nint a[N];\nmeta_schedule { meta_for (int i = 0; i < N; i++) a[i] = 3 $ 4; }\n",  # bad character
    "int N;\nint a[N];\nmeta_schedule { meta_for (int i = 0; i < N; i++) if (a[i]) a[i] = 0; }\n",  # no comparison
    "int N;\nint a[N];\nmeta_schedule { @warp meta_for (int i = 0; i < N; i++) a[i] = 0; }\n",  # unknown annotation
    "int N;\nint a[N];\nmeta_schedule { meta_for (int i = 0; i < N; j++) a[i] = 0; }\n",      # wrong increment
    "int N;\nint a[N];\nmeta_schedule { meta_for (int i = 0; j < N; i++) a[i] = 0; }\n",      # wrong test
    "int N;\nint a[N];\nmeta_schedule { for (int i = 0; i < N; i++) a[i] = 0; }\n",           # no meta_for
    "int N;\nint a[N];\nmeta_schedule { meta_for (int i = 0; i < N; i++) meta_schedule { } }\n",
    "int N;\nint a[N];\nint b = ;\nmeta_schedule { meta_for (int i = 0; i < N; i++) a[i] = 0; }\n",
]

# three @grid loops: dsl.parse accepts it (the <= 2 rule is split_roles', which
# the interpreter never calls), and run_program runs it
HAND.append(("grid3", """int N;
int a[N];
int c[N * N * 2];
meta_schedule {
    @grid meta_for (int i = 0; i < N; i++)
    @grid meta_for (int j = 0; j < N; j++)
    @grid meta_for (int k = 0; k < 2; k++)
        c[(i * N + j) * 2 + k] = a[i] - a[j] * k;
}
""", {"N": 6}))

# one 4-deep annotated program that is valid, and one with 2 grid / 2 thread loops by position
HAND.append(("annot4", """int N, M;
int a[N][M];
int c[N][M];
meta_schedule {
    @grid meta_for (int i = 0; i < N; i++)
    @thread meta_for (int j = 0; j < M; j++)
    @thread meta_for (int k = 0; k < 1; k++)
        c[i][j] = a[i][j] * 2 - k;
}
""", {"N": 5, "M": 6}))


def value_inputs(rng, prog, params, style):
    """Seeded arrays for every declared 1-D / 2-D array of ``prog`` (parakern)."""
    from parakern import interp

    shapes = {}
    m = interp.Machine(prog, dict(params))
    for name, data in m.arrays.items():
        shapes[name] = (len(data), len(data[0])) if data and isinstance(data[0], list) else (len(data),)

    def val():
        if style == "int":
            return rng.randint(-60, 60)
        if style == "wide":
            return rng.choice([rng.randint(-2**62, 2**62), rng.randint(-5, 5), 2**63 - 1, -2**63])
        if style == "float":
            return rng.choice([rng.uniform(-100, 100), float(rng.randint(-9, 9)), -0.0, 0.1, 1e308, -1e-310,
                               float("inf")])
        if style == "mixed":
            return rng.choice([rng.randint(-20, 20), rng.uniform(-5, 5), True, False])
        return rng.choice([rng.randint(-3, 3), "s%d" % rng.randint(0, 9), None, (1, 2), 2.5, False])

    out = {}
    for name, shp in shapes.items():
        if name.startswith("c"):
            continue  # outputs start as zeros (not supplied) in half the runs
        if len(shp) == 1:
            out[name] = [val() for _ in range(shp[0])]
        else:
            out[name] = [[val() for _ in range(shp[1])] for _ in range(shp[0])]
    return out


def structure(prog):
    from parakern import dsl

    try:
        grid, thread = dsl.split_roles(prog)
    except dsl.DslError:  # more than two grid or thread loops: roles as annotated
        grid = tuple(m for m in prog.meta_loops() if m.role == "grid")
        thread = tuple(m for m in prog.meta_loops() if m.role == "thread")
    scalars = [n for d in prog.decls if isinstance(d, dsl.ScalarDecl) for n in d.names]
    return {"scalars": scalars, "arrays": {n: [dsl.render_expr(x) for x in d.dims] for n, d in prog.arrays().items()},
            "bindings": [b.name for b in prog.bindings()], "context": [c.var for c in prog.context_loops],
            "meta": [m.var for m in prog.meta_loops()], "grid": [m.var for m in grid],
            "thread": [m.var for m in thread]}


def run(prog, params, arrays):
    from parakern import interp

    try:
        return {"outputs": interp.run_program(prog, dict(params), arrays=json.loads(json.dumps(arrays)))}
    except (IndexError, ZeroDivisionError, KeyError, TypeError) as exc:
        return {"error": type(exc).__name__}


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    args = ap.parse_args()
    sys.path.insert(0, args.ref)
    from parakern import dsl

    rng = random.Random(0x6E4)
    programs = [(name, text, params) for name, text, params in HAND]
    for k in range(48):
        shape = ["map1d", "map2d", "stencil", "triangle"][k % 4]
        text, params = generic_programs.program(rng, shape, safe_div=(k % 5 != 0), oob=(k % 7 == 3 and
                                                                                      shape != "stencil"))
        programs.append(("rand%02d_%s" % (k, shape), text, params))
    vectors, rejected = [], []
    for name, text, params in programs:
        prog = dsl.parse(text)
        entry = {"name": name, "text": text, "params": params, "structure": structure(prog), "runs": []}
        styles = ["int", "wide", "float", "mixed"] + (["objects"] if name == "move" else [])
        for style in styles:
            arrays = value_inputs(rng, prog, params, style)
            if style == "objects":  # objects are not JSON: tuples / None stand in as their repr
                arrays = {k: [v if isinstance(v, (int, float, str)) else repr(v) for v in vs] for k, vs in arrays.items()}
            r = run(prog, params, arrays)
            r.update({"style": style, "inputs": arrays})
            entry["runs"].append(r)
        # zeros only (no arrays supplied), and a missing parameter
        entry["runs"].append(dict(run(prog, params, {}), style="none", inputs={}))
        if params:
            drop = sorted(params)[0]
            p2 = {k: v for k, v in params.items() if k != drop}
            try:
                from parakern import interp

                interp.run_program(prog, p2)
                entry["missing_param"] = None
            except KeyError:
                entry["missing_param"] = {"drop": drop, "error": "KeyError"}
        # run_block (interp.py:228-249): grid values fixed, thread loops swept
        try:
            grid, _ = dsl.split_roles(prog)
        except dsl.DslError:
            grid = None
        if grid is not None and len(vectors) < 40:
            from parakern import interp

            entry["blocks"] = []
            arrays = value_inputs(rng, prog, params, "int")
            for pick in ("zero", "inside", "past"):
                gv = {}
                for m in grid:
                    bound = interp.Machine(prog, dict(params)).eval(m.bound) if not any(
                        x.var in dsl._names_in(m.bound) for x in prog.meta_loops()) else 1
                    gv[m.var] = {"zero": 0, "inside": rng.randrange(max(bound, 1)), "past": max(bound, 0) + 1}[pick]
                cv = {c.var: rng.randrange(2) for c in prog.context_loops}
                try:
                    out = interp.run_block(prog, dict(params), gv, cv, arrays=json.loads(json.dumps(arrays)))
                    res = {"outputs": out}
                except (IndexError, ZeroDivisionError, KeyError, TypeError) as exc:
                    res = {"error": type(exc).__name__}
                entry["blocks"].append(dict(res, grid_values=gv, context_values=cv, inputs=arrays))
        vectors.append(entry)
    for text in BAD:
        try:
            dsl.parse(text)
            raise SystemExit("expected a DslError for:\n" + text)
        except dsl.DslError as exc:
            rejected.append({"text": text, "error": str(exc)})
    out = os.path.join(HERE, "generic_vectors.json")
    with open(out, "w") as fh:
        json.dump({"generator": "parakern.dsl.parse + parakern.interp.run_program via tests/golden/make_generic.py",
                   "seed": "0x6E4", "programs": vectors, "rejected": rejected}, fh, separators=(",", ":"))
        fh.write("\n")
    print("wrote", out, len(vectors), "programs", sum(len(v["runs"]) for v in vectors), "runs", len(rejected),
          "rejected", os.path.getsize(out), "bytes")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
