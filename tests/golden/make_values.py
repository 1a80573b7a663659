"""Generate tests/golden/value_vectors.json from the REFERENCE interpreter:
values beyond the 32-bit words of interp_vectors.json.

The reference interpreter stores Python objects (interp.py:76-81,
183-206): binary64 floats at full precision, ints of any size, and -- for the
programs that only move values -- whatever object the caller supplied.  This
script runs parakern.interp.run_program (/root/reference/pkg/src/parakern/
interp.py:215) on seeded instances of

* reverse / transpose with binary64 floats (full 53-bit mantissas, -0.0,
  subnormals, +-inf, 1e308), ints beyond int32 and int64, bools and mixed
  int / float lists;
* addition / matvec / matmul with binary64 floats (the executor's
  PK_DTYPE_F64 path must reproduce them bit for bit) and with ints whose
  results leave int32 (the int64 path) or int64 (recorded: the executor
  raises OverflowError there);

and records inputs and outputs.  Only this script touches /root/reference.

    python tests/golden/make_values.py [--ref /root/reference/pkg/src]
"""

from __future__ import annotations

import argparse
import itertools
import json
import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

SPECIALS = [0.0, -0.0, 5e-324, -2.2250738585072014e-308, 1e308, -1.7976931348623157e308,
            float("inf"), float("-inf"), 0.1, 1 / 3]


def value(style: str, rng: random.Random):
    if style == "f64":
        r = rng.random()
        if r < 0.15:
            return rng.choice(SPECIALS)
        return rng.uniform(-1.0, 1.0) * 10.0 ** rng.randrange(-30, 30)
    if style == "f64_unit":
        return rng.uniform(-1.0, 1.0)
    if style == "i64":
        return rng.randrange(-(2**62), 2**62)
    if style == "bigint":
        return rng.randrange(-(2**90), 2**90)
    if style == "mixed":
        return rng.choice([rng.randrange(-(2**40), 2**40), rng.uniform(-5, 5), True, False, 7])
    if style == "i_wide":  # arithmetic: results leave int32, stay in int64
        return rng.randrange(-(2**26), 2**26)
    if style == "i_huge":  # arithmetic: results leave int64
        return rng.randrange(-(2**40), 2**40)
    raise KeyError(style)


def fill(shape, style, rng):
    if len(shape) == 1:
        return [value(style, rng) for _ in range(shape[0])]
    return [fill(shape[1:], style, rng) for _ in range(shape[0])]


PARAMS = {
    "reverse": [{"N": 64, "s": 2, "B": 8}, {"N": 37, "s": 2, "B": 8}, {"N": 16, "s": 1, "B": 4}],
    "transpose": [{"N": 16, "s": 2, "B0": 4, "B1": 2}, {"N": 7, "s": 2, "B0": 3, "B1": 2}],
    "addition": [{"N": 8, "B0": 2, "B1": 2}, {"N": 6, "B0": 4, "B1": 1}],
    "matvec": [{"N": 16, "s": 2, "B": 4}, {"N": 11, "s": 2, "B": 3}],
    "matmul": [{"n": 12, "B0": 4, "ub1": 2, "s": 2}, {"n": 10, "B0": 3, "ub1": 2, "s": 2}],
}
STYLES = {
    "reverse": ["f64", "i64", "bigint", "mixed"],
    "transpose": ["f64", "i64", "bigint", "mixed"],
    "addition": ["f64", "f64_unit", "i_wide", "i_huge"],
    "matvec": ["f64", "f64_unit", "i_wide", "i_huge"],
    "matmul": ["f64_unit", "f64", "i_wide", "i_huge"],
}


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    args = ap.parse_args()
    sys.dont_write_bytecode = True
    sys.path.insert(0, args.ref)
    from parakern import dsl, interp  # noqa: E402

    from paper_1801_04348_b200 import programs  # noqa: E402

    rng = random.Random(0x64F)
    vectors = []
    for family in sorted(PARAMS):
        prog = dsl.parse(programs.original(family).text)
        for params in PARAMS[family]:
            for style in STYLES[family]:
                shapes = {}
                for name, data in interp.Machine(prog, dict(params)).arrays.items():
                    shapes[name] = (len(data), len(data[0])) if data and isinstance(data[0], list) else (len(data),)
                seed = {name: fill(shape, style, rng) for name, shape in shapes.items()}
                if family in ("reverse", "transpose") and style != "mixed":
                    seed.pop("c")  # the unwritten part of c stays int 0 (interp.py:79-81)
                want = interp.run_program(prog, dict(params), arrays=seed)
                vectors.append({"family": family, "params": params, "style": style, "inputs": seed,
                                "outputs": want})
    # the stencils on binary64 floats (c_div on Python floats) and on ints
    # beyond int32, whole programs
    for family, params in [("jacobi", {"T": 4, "N": 26, "s": 2, "B": 4}), ("jacobi", {"T": 3, "N": 19, "s": 3, "B": 2}),
                           ("jacobi2d", {"T": 3, "N": 11, "s": 2, "B0": 2, "B1": 2})]:
        prog = dsl.parse(programs.original(family).text)
        for style in ("f64", "f64_unit", "i64"):
            shapes = {}
            for name, data in interp.Machine(prog, dict(params)).arrays.items():
                shapes[name] = (len(data), len(data[0])) if data and isinstance(data[0], list) else (len(data),)
            seed = {name: fill(shape, style, rng) for name, shape in shapes.items()}
            if style == "i64":  # sums of 5 stay in int64
                seed = {k: [[x // 8 for x in r] for r in v] if v and isinstance(v[0], list) else [x // 8 for x in v]
                        for k, v in seed.items()}
            want = interp.run_program(prog, dict(params), arrays=seed)
            vectors.append({"family": family, "params": params, "style": style, "inputs": seed, "outputs": want})
    # run_block (interp.py:228-249) on values beyond 32-bit words: every grid
    # point of small instances, original programs and their granularity case
    # programs, binary64 floats and wide ints
    from parakern import model, strategies  # noqa: E402

    blocks = []
    BLOCK_PARAMS = {"jacobi": {"T": 3, "N": 26, "s": 2, "B": 4}, "jacobi2d": {"T": 2, "N": 11, "s": 2, "B0": 2, "B1": 2},
                    "reverse": {"N": 37, "s": 2, "B": 4}, "transpose": {"N": 9, "s": 2, "B0": 2, "B1": 2},
                    "matvec": {"N": 11, "s": 2, "B": 3}, "matmul": {"n": 8, "B0": 2, "ub1": 2, "s": 2},
                    "addition": {"N": 8, "B0": 2, "B1": 2}}
    for family in sorted(BLOCK_PARAMS):
        a = BLOCK_PARAMS[family]
        prog = dsl.parse(programs.original(family).text)
        cfg = model.build_source_cfg(prog)
        m = interp.Machine(prog, dict(a))
        grid = [(gv.var, m.eval(gv.bound)) for gv in cfg.grid]
        context = [(cv.var, m.eval(cv.bound)) for cv in cfg.context]
        shapes = {}
        for name, data in m.arrays.items():
            shapes[name] = (len(data), len(data[0])) if data and isinstance(data[0], list) else (len(data),)
        for style in ("f64", "i64"):
            seed = {name: fill(shape, style, rng) for name, shape in shapes.items()}
            if style == "i64":
                seed = {k: [[x >> 40 for x in r] for r in v] if v and isinstance(v[0], list) else [x >> 40 for x in v]
                        for k, v in seed.items()}  # |v| < 2^22: products and sums stay in int64
            ctx = {v: rng.randrange(max(1, b)) for v, b in context}
            for point in itertools.product(*[range(b) for _, b in grid]):
                gv = {v: p for (v, _), p in zip(grid, point)}
                want = interp.run_block(prog, dict(a), gv, dict(ctx), arrays=seed)
                blocks.append({"family": family, "style": style, "program": "original", "params": a,
                               "grid_values": gv, "context_values": ctx, "inputs": seed, "outputs": want})
            # one grid point past the meta_for range: the reference raises IndexError
            gv = {v: b for v, b in grid}
            try:
                interp.run_block(prog, dict(a), gv, dict(ctx), arrays=seed)
                err = None
            except IndexError:
                err = "IndexError"
            blocks.append({"family": family, "style": style, "program": "original", "params": a, "grid_values": gv,
                           "context_values": ctx, "inputs": seed, "error": err})
        # the granularity case program (s removed, s := 1), one grid point
        try:
            gp = strategies.apply_source("granularity", prog)
        except ValueError:
            continue
        ga = {k: v for k, v in a.items() if k != "s"}
        gm = interp.Machine(gp, dict(ga))
        gcfg = model.build_source_cfg(gp)
        ggrid = {gv.var: 0 for gv in gcfg.grid}
        gctx = {cv.var: 0 for cv in gcfg.context}
        gshapes = {n: ((len(d), len(d[0])) if d and isinstance(d[0], list) else (len(d),)) for n, d in gm.arrays.items()}
        seed = {name: fill(shape, "f64", rng) for name, shape in gshapes.items()}
        want = interp.run_block(gp, dict(ga), ggrid, dict(gctx), arrays=seed)
        blocks.append({"family": family, "style": "f64", "program": dsl.render(gp), "params": ga,
                       "grid_values": ggrid, "context_values": gctx, "inputs": seed, "outputs": want})
    # IndexError (interp.py:209-212): the shortest 1-D array each program runs
    # on without an out-of-bounds access -- what pk_required_elems must report
    bounds = []
    for family, params in [("reverse", {"N": 100, "s": 2, "B": 32}), ("reverse", {"N": 64, "s": 1, "B": 8}),
                           ("matvec", {"N": 10, "s": 1, "B": 4}), ("matvec", {"N": 9, "s": 2, "B": 2}),
                           ("jacobi", {"T": 1, "N": 10, "s": 2, "B": 2}),
                           ("jacobi", {"T": 3, "N": 12, "s": 1, "B": 3})]:
        prog = dsl.parse(programs.original(family).text)
        full = interp.Machine(prog, dict(params)).arrays
        mins = {}
        for name, data in full.items():
            if data and isinstance(data[0], list):
                continue
            n = len(data)
            while n > 0:
                arrays = {k: (list(v) if k != name else [0] * (n - 1)) for k, v in full.items()}
                try:
                    interp.run_program(prog, dict(params), arrays=arrays)
                except IndexError:
                    break
                n -= 1
            mins[name] = n
        bounds.append({"family": family, "params": params, "min_len": mins})
    out = os.path.join(HERE, "value_vectors.json")
    with open(out, "w") as fh:
        json.dump({"generator": "parakern.interp.run_program via tests/golden/make_values.py",
                   "seed": "0x64F", "vectors": vectors, "bounds": bounds, "blocks": blocks}, fh,
                  separators=(",", ":"))
        fh.write("\n")
    print("wrote", out, len(vectors), "vectors", os.path.getsize(out), "bytes")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
