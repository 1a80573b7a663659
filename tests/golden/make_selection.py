"""Generate tests/golden/case_selection.json from the REFERENCE engine.

For every program family and both machine models, runs
``parakern.engine.optimize`` and records, at sampled points (program
parameters + machine values), which cases' systems hold according to the
reference's own ``ConstraintSystem.holds`` (algebra.py:621-622).  The shipped
evaluator (paper_1801_04348_b200/cases.py) must reproduce these exactly.

    python tests/golden/make_selection.py [--ref /root/reference/pkg/src]
"""

from __future__ import annotations

import argparse
import json
import os
import random
import sys
from fractions import Fraction

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

MACHINE_POINTS = {
    "fermi": [{"Z_B": 12288, "R_B": 63}, {"Z_B": 300, "R_B": 63}, {"Z_B": 12288, "R_B": 10},
              {"Z_B": 40, "R_B": 6}],
    "b200": [{"Z_B": 58112, "R_B": 255, "T_B": 1024}, {"Z_B": 12288, "R_B": 255, "T_B": 1024},
             {"Z_B": 4000, "R_B": 8, "T_B": 1024}, {"Z_B": 58112, "R_B": 255, "T_B": 256}],
    # occupancy model: R_F = the register file, O = the target ratio (as a string)
    "b200-occ": [{"Z_B": 58112, "R_B": 255, "T_B": 1024, "R_F": 65536, "O": "1"},
                 {"Z_B": 58112, "R_B": 255, "T_B": 1024, "R_F": 65536, "O": "1/2"},
                 {"Z_B": 12288, "R_B": 255, "T_B": 1024, "R_F": 65536, "O": "1/8"},
                 {"Z_B": 58112, "R_B": 8, "T_B": 1024, "R_F": 32768, "O": "3/4"}],
}


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    args = ap.parse_args()
    sys.dont_write_bytecode = True
    sys.path.insert(0, args.ref)
    from parakern import dsl, engine
    from parakern.machine import load_machine

    from paper_1801_04348_b200 import programs

    ref_data = os.path.join(args.ref, "parakern", "data")
    machines = {
        "fermi": load_machine(os.path.join(ref_data, "fermi.machine")),
        "addition-target": load_machine(os.path.join(ref_data, "addition.machine")),
        "b200": load_machine(os.path.join(REPO, "paper_1801_04348_b200", "data", "b200.machine")),
        "b200-occ": load_machine(os.path.join(REPO, "paper_1801_04348_b200", "data", "b200-occ.machine")),
    }
    rng = random.Random(0xCA5E)
    records = []
    for family in sorted(programs.FAMILIES):
        prog = dsl.parse(programs.original(family).text)
        for mname in ("fermi", "b200"):
            m = machines["addition-target" if (family == "addition" and mname == "fermi") else mname]
            result = engine.optimize(prog, m)
            names = list(result.table.order)
            for _ in range(60):
                point = {}
                for n in names:
                    lo, hi = result.box[n]
                    hi = min(int(hi), 4096 if n in ("N", "n") else int(hi))
                    point[n] = rng.randint(int(lo), hi)
                mp = dict(rng.choice(MACHINE_POINTS[mname]))
                if family == "addition" and mname == "fermi":
                    mp = {"T_B": 1024, "R_B": rng.choice([63, 4, 5])}
                assignment = {k: Fraction(v) for k, v in {**point, **mp}.items()}
                holding = [c.index for c in result.cases if c.system.holds(assignment)]
                records.append({"family": family, "machine": result.machine.name, "params": point,
                                "machine_values": mp, "holding": holding})
    # the occupancy model (separate stream, so the records above stay as they were)
    rng = random.Random(0x0CC)
    for family in sorted(programs.FAMILIES):
        prog = dsl.parse(programs.original(family).text)
        result = engine.optimize(prog, machines["b200-occ"])
        names = list(result.table.order)
        for _ in range(60):
            point = {}
            for n in names:
                lo, hi = result.box[n]
                hi = min(int(hi), 4096 if n in ("N", "n") else int(hi))
                point[n] = rng.randint(int(lo), hi)
            mp = dict(rng.choice(MACHINE_POINTS["b200-occ"]))
            assignment = {k: Fraction(v) for k, v in {**point, **mp}.items()}
            holding = [c.index for c in result.cases if c.system.holds(assignment)]
            records.append({"family": family, "machine": result.machine.name, "params": point,
                            "machine_values": mp, "holding": holding})
    out = os.path.join(HERE, "case_selection.json")
    with open(out, "w") as fh:
        json.dump({"generator": "parakern ConstraintSystem.holds via tests/golden/make_selection.py",
                   "records": records}, fh, separators=(",", ":"))
        fh.write("\n")
    print("wrote", out, len(records), "records")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
