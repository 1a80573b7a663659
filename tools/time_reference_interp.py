"""Time the reference's own CPU path -- parakern.interp.run_program, the
pure-Python interpreter this executor replaces -- at the reduced instances
of SURVEY.md 8(d) / BASELINE.md 3, one core, and write
profiles/r02_reference_interp.json.

The reference cannot travel to the GPU box (nothing there may read
/root/reference), so its rate is measured here, in the build container, and
bench.py reports it beside the oracle port it times on the box's own cores.
Rates are per unit of the bench's metric (bytes of algorithmic traffic for
the bandwidth families, FLOP for matmul) so they compare with the GPU line
directly, plus the interpreter's own points (or FMAs) per second.

    python tools/time_reference_interp.py [--ref /root/reference/pkg/src]
"""

from __future__ import annotations

import argparse
import json
import os
import platform
import random
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

# family: (params, points the program updates, algorithmic work, unit) -- SURVEY 8(d) reduced instances
INSTANCES = {
    "reverse": ({"N": 1 << 16, "s": 4, "B": 64}, 1 << 16, 8 * (1 << 16), "B"),
    "transpose": ({"N": 256, "s": 4, "B0": 16, "B1": 4}, 256 * 256, 8 * 256 * 256, "B"),
    "jacobi": ({"T": 4, "N": (1 << 14) + 2, "s": 4, "B": 64}, 4 * (1 << 14), 4 * 8 * (1 << 14), "B"),
    "jacobi2d": ({"T": 2, "N": 130, "s": 2, "B0": 8, "B1": 16}, 2 * 128 * 128, 2 * 8 * 128 * 128, "B"),
    "matvec": ({"N": 256, "s": 1, "B": 32}, 256 * 256, 4 * 256 * 256 + 8 * 256, "B"),
    "matmul": ({"n": 48, "B0": 16, "ub1": 4, "s": 3}, 48 ** 3, 2 * 48 ** 3, "FLOP"),
}


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    ap.add_argument("--out", default=os.path.join(REPO, "profiles", "r02_reference_interp.json"))
    args = ap.parse_args()
    sys.dont_write_bytecode = True
    sys.path.insert(0, args.ref)
    from parakern import dsl, interp  # noqa: E402

    from paper_1801_04348_b200 import programs  # noqa: E402

    rng = random.Random(0x1801)
    out = {}
    for fam, (params, points, work, unit) in INSTANCES.items():
        prog = dsl.parse(programs.original(fam).text)
        seed = {}
        for name, data in interp.Machine(prog, dict(params)).arrays.items():
            if data and isinstance(data[0], list):
                seed[name] = [[rng.randrange(-50, 50) for _ in row] for row in data]
            else:
                seed[name] = [rng.randrange(-50, 50) for _ in data]
        t0 = time.perf_counter()
        interp.run_program(prog, dict(params), arrays=seed)
        sec = time.perf_counter() - t0
        scale = 1e9
        out[fam] = {"params": params, "seconds": round(sec, 3), "points_per_s": round(points / sec, 1),
                    "value": round(work / sec / scale, 6),
                    "unit": "GB/s" if unit == "B" else "GFLOP/s", "cores": 1}
        print(fam, out[fam], flush=True)
    doc = {"what": "parakern.interp.run_program (the reference's CPU path), pure Python, 1 core",
           "where": "build container (no GPU): %s, Python %s" % (platform.processor() or platform.machine(),
                                                                 platform.python_version()),
           "script": "tools/time_reference_interp.py", "families": out}
    with open(args.out, "w") as fh:
        json.dump(doc, fh, indent=1)
        fh.write("\n")
    print("wrote", args.out)
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
