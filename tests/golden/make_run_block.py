"""Generate tests/golden/run_block_vectors.json from the REFERENCE interpreter.

Runs parakern.interp.run_block (/root/reference/pkg/src/parakern/interp.py:228-249)
-- one thread block: grid indices fixed, context loop variables supplied,
thread loops swept -- on small seeded instances of the seven program
families (original program and the caching-off case program), at every grid
point of the block grid for a random context value.  Only this script
touches /root/reference; the fixture travels.  Re-run from the repo root:

    python tests/golden/make_run_block.py [--ref /root/reference/pkg/src]
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
sys.path.insert(0, HERE)

PARAMS = {
    "jacobi": [{"T": 3, "N": 26, "s": 2, "B": 4}, {"T": 2, "N": 19, "s": 3, "B": 2}],
    "jacobi2d": [{"T": 2, "N": 11, "s": 2, "B0": 2, "B1": 2}],
    "reverse": [{"N": 37, "s": 2, "B": 4}],
    "transpose": [{"N": 9, "s": 2, "B0": 2, "B1": 2}],
    "matvec": [{"N": 11, "s": 2, "B": 3}],
    "matmul": [{"n": 8, "B0": 2, "ub1": 2, "s": 2}],
    "addition": [{"N": 8, "B0": 2, "B1": 2}],
}


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    args = ap.parse_args()
    sys.dont_write_bytecode = True
    sys.path.insert(0, args.ref)
    from make_golden import fill  # noqa: E402
    from parakern import dsl, interp, model, strategies  # noqa: E402

    from paper_1801_04348_b200 import programs  # noqa: E402

    rng = random.Random(0x1801 + 7)
    vectors = []
    for family in sorted(PARAMS):
        prog = dsl.parse(programs.original(family).text)
        variants = [("original", prog)]
        try:
            variants.append(("caching-off", strategies.apply_source("caching-off", prog)))
        except ValueError:  # nothing cached (addition)
            pass
        for a in PARAMS[family]:
            cfg = model.build_source_cfg(prog)
            m = interp.Machine(prog, dict(a))
            grid = [(g.var, m.eval(g.bound)) for g in cfg.grid]
            context = [(c.var, m.eval(c.bound)) for c in cfg.context]
            shapes = {}
            for name, data in m.arrays.items():
                shapes[name] = (len(data), len(data[0])) if data and isinstance(data[0], list) else (len(data),)
            for vname, vprog in variants:
                seed = {name: fill(shape, rng) for name, shape in shapes.items()}
                ctx = {v: rng.randrange(max(1, b)) for v, b in context}
                for point in itertools.product(*[range(b) for _, b in grid]):
                    gv = {v: p for (v, _), p in zip(grid, point)}
                    want = interp.run_block(vprog, dict(a), gv, dict(ctx), arrays=seed)
                    vectors.append({"family": family, "variant": vname, "program": dsl.render(vprog),
                                    "params": a, "grid_values": gv, "context_values": ctx,
                                    "inputs": seed, "outputs": want})
    out = os.path.join(HERE, "run_block_vectors.json")
    with open(out, "w") as fh:
        json.dump({"generator": "parakern.interp.run_block via tests/golden/make_run_block.py",
                   "vectors": vectors}, fh, separators=(",", ":"))
        fh.write("\n")
    print("wrote", out, len(vectors), "vectors", os.path.getsize(out), "bytes")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
