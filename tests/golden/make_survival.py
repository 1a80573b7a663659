"""Generate tests/golden/survival.json with the REFERENCE's consistency
checker: for every shipped case table and machine model, which leaves can
hold once the machine parameters are fixed (the live B200 values, its 48 KB
static carve-out, the occupancy model at O = 1/2, and the reference's Fermi
limits).  Uses parakern.algebra.check_consistency
(/root/reference/pkg/src/parakern/algebra.py:722-911) on each leaf's system
with the machine values substituted (the _machine_feasible pattern,
engine.py:514-528, roles swapped: machine fixed, program parameters free in
the table's box).  Only this script touches /root/reference.

    python tests/golden/make_survival.py [--ref /root/reference/pkg/src]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
from fractions import Fraction

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    args = ap.parse_args()
    sys.dont_write_bytecode = True
    sys.path.insert(0, args.ref)
    from parakern.algebra import Constraint, ConstraintSystem, Poly, check_consistency  # noqa: E402

    from paper_1801_04348_b200 import cases, machine, programs  # noqa: E402

    models = {
        "b200": machine.nominal(),
        "b200-static": machine.nominal(smem="static"),
        "b200-occ": machine.nominal(occupancy=Fraction(1, 2)),
        "fermi": machine.fermi(),
    }
    out = []
    for family in sorted(programs.FAMILIES):
        for label, mv in models.items():
            try:
                tab = cases.table(family, mv.table)
            except KeyError:
                continue
            with open(os.path.join(REPO, "paper_1801_04348_b200", "data", "cases",
                                   "%s.%s.json" % (family, tab.machine if tab.machine != "fermi" or family != "addition"
                                                   else "addition-target"))) as fh:
                box = {k: (int(v[0]), int(v[1])) for k, v in json.load(fh)["box"].items()}
            fixed = {n: Fraction(mv.values[n]) for n in tab.machine_names()}
            pbox = {k: v for k, v in box.items() if k not in fixed}
            verdicts = []
            for case in tab.cases:
                cons = []
                for c in case.constraints:
                    terms = {}
                    for coeff, mono in c.poly:
                        terms[tuple(sorted(mono))] = terms.get(tuple(sorted(mono)), Fraction(0)) + Fraction(coeff)
                    p = Poly(terms).subs(fixed)
                    cons.append(Constraint(p, c.rel, Poly.const(0), c.initial))
                v = check_consistency(ConstraintSystem(cons), pbox)
                verdicts.append({"case": case.index, "status": v.status, "reason": v.reason})
            out.append({"family": family, "model": label, "table": tab.machine,
                        "values": {k: str(v) for k, v in fixed.items()}, "verdicts": verdicts})
            print(family, label, [(d["case"], d["status"]) for d in verdicts], flush=True)
    path = os.path.join(HERE, "survival.json")
    with open(path, "w") as fh:
        json.dump({"generator": "parakern.algebra.check_consistency via tests/golden/make_survival.py",
                   "tables": out}, fh, indent=1)
        fh.write("\n")
    print("wrote", path)
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
