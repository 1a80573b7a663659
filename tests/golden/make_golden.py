"""Generate tests/golden/interp_vectors.json from the REFERENCE interpreter.

Runs parakern.interp.run_program (/root/reference/pkg/src/parakern/interp.py:215)
on small seeded instances of every program family -- the original program
and, per the reference's c07 acceptance property
(pkg/tests/test_acceptance.py:433-458), every case program of its case
discussion under the parity-preserving parameter map -- and records inputs
and outputs.  Only this script touches /root/reference; the fixtures it
writes are what travels.  Re-run from the repo root:

    python tests/golden/make_golden.py [--ref /root/reference/pkg/src]
"""

from __future__ import annotations

import argparse
import json
import os
import random
import struct
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)


def f32(x: float) -> float:
    return struct.unpack("f", struct.pack("f", x))[0]


def granularity_map(family: str, a: dict) -> dict:
    """Parity-preserving parameters for a granularity case program
    (pkg/tests/test_acceptance.py:400-408, SURVEY App. A.1 for matmul)."""
    a = dict(a)
    if family in ("jacobi", "reverse", "matvec"):
        a["B"] = a["s"] * a["B"]
        a.pop("s")
    elif family in ("transpose", "jacobi2d"):
        a["B1"] = a["s"] * a["B1"]
        a.pop("s")
    elif family == "matmul":
        a["ub1"] = a["s"] * a["ub1"]
        a.pop("s")
    elif family == "addition":
        a["B1"] = 2 * a["B1"]
    return a


def sample(family: str, rng: random.Random) -> dict:
    r = rng.randrange
    if family == "jacobi":
        return {"T": r(1, 5), "N": r(4, 41), "s": r(1, 5), "B": r(1, 9)}
    if family == "transpose":
        return {"N": r(2, 17), "s": r(1, 4), "B0": r(1, 6), "B1": r(1, 6)}
    if family == "reverse":
        return {"N": r(1, 65), "s": r(1, 5), "B": r(1, 9)}
    if family == "matvec":
        return {"N": r(1, 17), "s": r(1, 4), "B": r(1, 6)}
    if family == "matmul":
        return {"n": r(1, 13), "B0": r(1, 5), "ub1": r(1, 4), "s": r(1, 4)}
    if family == "jacobi2d":
        return {"T": r(1, 4), "N": r(3, 13), "s": r(1, 3), "B0": r(1, 5), "B1": r(1, 4)}
    B1 = r(1, 5)
    return {"N": 2 * B1 * r(1, 5), "B0": r(1, 6), "B1": B1}


def fill(shape, rng, floats=False):
    if len(shape) == 1:
        if floats:
            return [f32(rng.uniform(-1.0, 1.0)) for _ in range(shape[0])]
        return [rng.randrange(-50, 50) for _ in range(shape[0])]
    return [fill(shape[1:], rng, floats) for _ in range(shape[0])]


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    args = ap.parse_args()
    sys.dont_write_bytecode = True
    sys.path.insert(0, args.ref)
    from parakern import dsl, interp  # noqa: E402

    from paper_1801_04348_b200 import cases, programs  # noqa: E402

    rng = random.Random(0x1801)
    vectors = []
    for family in sorted(programs.FAMILIES):
        kind = programs.original(family)
        prog = dsl.parse(kind.text)
        case_progs = {}
        for mname in ("fermi", "b200"):
            for c in cases.table(family, mname).cases:
                case_progs.setdefault(programs.normalize(c.program), (c.program, c.source_applied))
        n_vec = 14
        for i in range(n_vec):
            a = sample(family, rng)
            floats = family in ("matmul", "matvec") and i % 2 == 1
            machine_arrays = interp.Machine(prog, dict(a)).arrays
            shapes = {}
            for name, data in machine_arrays.items():
                shapes[name] = (len(data), len(data[0])) if data and isinstance(data[0], list) else (len(data),)
            seed = {name: fill(shape, rng, floats) for name, shape in shapes.items()}
            want = interp.run_program(prog, dict(a), arrays=seed)
            checked = []
            for text, applied in case_progs.values():
                if not applied:
                    continue
                cp = dsl.parse(text)
                mapped = granularity_map(family, a) if "granularity" in applied else dict(a)
                got = interp.run_program(cp, mapped, arrays=seed)
                assert got == want, (family, applied, a)
                checked.append(list(applied))
            vectors.append({"family": family, "program": "original", "params": a, "inputs": seed,
                            "outputs": want, "case_programs_checked": checked, "floats": floats})
        # the case programs themselves, run with their own parameters
        for text, applied in case_progs.values():
            if not applied:
                continue
            a = sample(family, rng)
            mapped = granularity_map(family, a) if "granularity" in applied else dict(a)
            cp = dsl.parse(text)
            machine_arrays = interp.Machine(cp, dict(mapped)).arrays
            seed = {}
            for name, data in machine_arrays.items():
                shape = (len(data), len(data[0])) if data and isinstance(data[0], list) else (len(data),)
                seed[name] = fill(shape, rng)
            want = interp.run_program(cp, dict(mapped), arrays=seed)
            vectors.append({"family": family, "program": text, "applied": list(applied),
                            "params": mapped, "inputs": seed, "outputs": want,
                            "case_programs_checked": [], "floats": False})
        # edge cases: tails, empty grids, zero divisors
        edges = {
            "jacobi": [{"T": 2, "N": 26, "s": 2, "B": 8}, {"T": 3, "N": 2, "s": 1, "B": 1},
                       {"T": 0, "N": 10, "s": 1, "B": 2}, {"T": 2, "N": 9, "s": 4, "B": 4}],
            "reverse": [{"N": 37, "s": 2, "B": 8}, {"N": 5, "s": 2, "B": 4}],
            "transpose": [{"N": 7, "s": 2, "B0": 3, "B1": 2}, {"N": 3, "s": 2, "B0": 4, "B1": 2}],
            "matvec": [{"N": 11, "s": 2, "B": 3}],
            "matmul": [{"n": 10, "B0": 3, "ub1": 2, "s": 2}, {"n": 7, "B0": 4, "ub1": 1, "s": 3}],
            "jacobi2d": [{"T": 3, "N": 11, "s": 2, "B0": 4, "B1": 2}],
            "addition": [{"N": 7, "B0": 2, "B1": 2}],
        }[family]
        for a in edges:
            machine_arrays = interp.Machine(prog, dict(a)).arrays
            seed = {}
            for name, data in machine_arrays.items():
                shape = (len(data), len(data[0])) if data and isinstance(data[0], list) else (len(data),)
                seed[name] = fill(shape, rng)
            want = interp.run_program(prog, dict(a), arrays=seed)
            vectors.append({"family": family, "program": "original", "params": a, "inputs": seed,
                            "outputs": want, "case_programs_checked": [], "floats": False, "edge": True})
        zero = {"jacobi": {"T": 1, "N": 6, "s": 0, "B": 2}, "reverse": {"N": 8, "s": 2, "B": 0},
                "transpose": {"N": 4, "s": 1, "B0": 0, "B1": 1}, "matvec": {"N": 4, "s": 0, "B": 1},
                "matmul": {"n": 4, "B0": 0, "ub1": 1, "s": 1},
                "jacobi2d": {"T": 1, "N": 5, "s": 1, "B0": 1, "B1": 0},
                "addition": {"N": 4, "B0": 1, "B1": 0}}[family]
        try:
            interp.run_program(prog, dict(zero))
            err = None
        except ZeroDivisionError:
            err = "ZeroDivisionError"
        vectors.append({"family": family, "program": "original", "params": zero, "error": err})

    out = os.path.join(HERE, "interp_vectors.json")
    with open(out, "w") as fh:
        json.dump({"generator": "parakern.interp.run_program via tests/golden/make_golden.py",
                   "seed": "0x1801", "vectors": vectors}, fh, separators=(",", ":"))
        fh.write("\n")
    print("wrote", out, len(vectors), "vectors", os.path.getsize(out), "bytes")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
