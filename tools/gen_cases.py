"""Regenerate the shipped case tables (paper_1801_04348_b200/data/cases/*.json).

The case discussion is the reference's LOAD-TIME product: it is built by
``parakern.engine.optimize`` (/root/reference/pkg/src/parakern/engine.py:495)
and is symbolic in the machine parameters (Z_B, R_B, T_B), so it is computed
once here, where the reference is importable, and shipped as data.  The
executor evaluates the stored constraint systems against the LIVE device
properties (``ConstraintSystem.holds``, algebra.py:621-622, restated in
paper_1801_04348_b200/cases.py).

Run from the repo root (needs /root/reference; NOT used at run time):

    python tools/gen_cases.py [--ref /root/reference/pkg/src]
"""

from __future__ import annotations

import argparse
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
PKG_DATA = os.path.join(REPO, "paper_1801_04348_b200", "data")

# family -> (program file, reference machine file for the "default machine")
FAMILIES = {
    "jacobi": ("ref:jacobi.mfk", "fermi.machine"),
    "transpose": ("ref:transpose.mfk", "fermi.machine"),
    "addition": ("ref:addition.mfk", "addition.machine"),
    "reverse": ("pkg:reverse.mfk", "fermi.machine"),
    "matvec": ("pkg:matvec.mfk", "fermi.machine"),
    "matmul": ("pkg:matmul.mfk", "fermi.machine"),
    "jacobi2d": ("pkg:jacobi2d.mfk", "fermi.machine"),
}


def _poly_json(poly):
    terms = []
    for mono, coeff in poly.sorted_terms():
        terms.append([str(coeff), [[n, e] for n, e in mono]])
    return terms


def _constraint_json(c, order):
    return {
        "rel": c.rel,
        "poly": _poly_json(c.poly),
        "initial": bool(c.initial),
        "text": c.text(order),
    }


def build(ref_src: str) -> dict:
    sys.path.insert(0, ref_src)
    from parakern import dsl, engine, emit  # noqa: F401
    from parakern.machine import load_machine

    ref_data = os.path.join(ref_src, "parakern", "data")
    machines = {
        "fermi.machine": load_machine(os.path.join(ref_data, "fermi.machine")),
        "addition.machine": load_machine(os.path.join(ref_data, "addition.machine")),
        "b200.machine": load_machine(os.path.join(PKG_DATA, "b200.machine")),
        "b200-occ.machine": load_machine(os.path.join(PKG_DATA, "b200-occ.machine")),
    }
    out = {}
    for fam, (prog_ref, default_machine) in FAMILIES.items():
        where, fname = prog_ref.split(":")
        base = ref_data if where == "ref" else os.path.join(PKG_DATA, "programs")
        with open(os.path.join(base, fname)) as fh:
            program = dsl.parse(fh.read())
        for mfile in (default_machine, "b200.machine", "b200-occ.machine"):
            machine = machines[mfile]
            result = engine.optimize(program, machine)
            order = result.order
            table = result.table
            cases = []
            for case in result.cases:
                ctable = dsl.classify_parameters(case.program)
                cases.append(
                    {
                        "index": case.index,
                        "applied": list(case.applied),
                        "trail": list(case.trail),
                        "program": dsl.render(case.program),
                        "params": list(ctable.order),
                        "constraints": [_constraint_json(c, order) for c in case.system],
                        "header": [
                            c.text(order)
                            for c in engine.case_header(case, result.box, order)
                        ],
                        "witness": {k: str(v) for k, v in sorted(case.witness.items())}
                        if case.witness
                        else None,
                    }
                )
            doc = {
                "family": fam,
                "machine": machine.name,
                "machine_file": mfile,
                "generated_by": "parakern.engine.optimize (reference engine.py:495)",
                "source": dsl.render(program),
                "order": list(order),
                "params": list(table.order),
                "data_params": list(table.data),
                "program_params": list(table.program),
                "machine_params": [
                    {"name": p.name, "kind": p.kind, "lo": str(p.lo), "hi": str(p.hi)}
                    for p in machine.params
                ],
                "counters": [
                    {"name": c.name, "measure": c.measure, "bound": c.bound, "kind": c.kind,
                     "options": dict(c.options)}
                    for c in machine.counters
                ],
                "box": {k: [str(v[0]), str(v[1])] for k, v in result.box.items()},
                "decision_height": result.tree.height(),
                "cases": cases,
                "tree": json.loads(emit.export_tree_json(result, name=fam)),
            }
            out[(fam, machine.name)] = doc
    return out


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    args = ap.parse_args()
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    sys.dont_write_bytecode = True
    docs = build(args.ref)
    dest = os.path.join(PKG_DATA, "cases")
    os.makedirs(dest, exist_ok=True)
    for (fam, mname), doc in sorted(docs.items()):
        path = os.path.join(dest, "%s.%s.json" % (fam, mname))
        with open(path, "w") as fh:
            json.dump(doc, fh, indent=1, sort_keys=True)
            fh.write("\n")
        print("wrote", os.path.relpath(path, REPO), len(doc["cases"]), "cases")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
