"""Case-tree evaluation against live machine parameters.

The case discussion (the leaves (C_i, S_i) of the reference's Algorithm 1,
engine.py:439-492) is symbolic in the machine parameters.  It is produced
at build time by the reference's own engine (tools/gen_cases.py) and loaded
here; at run time each leaf's constraint system is evaluated EXACTLY
(rational arithmetic) at program parameters + live device values:

* ``Poly.eval``             algebra.py:161-169   -> :func:`_eval_poly`
* ``Constraint.holds``      algebra.py:507-513   -> :meth:`Constraint.holds`
* ``ConstraintSystem.holds`` algebra.py:621-622  -> :meth:`Case.holds`

Sibling edges carry complementary constraints (engine.py:372-379), so at a
point inside the box exactly one case holds; :func:`select` returns it.
"""

from __future__ import annotations

import json
import os
from dataclasses import dataclass
from fractions import Fraction
from functools import lru_cache

from . import machine as machine_mod
from .programs import DATA, SOURCE_STRATEGIES, ProgramKind


def _eval_poly(terms, assignment) -> Fraction:
    total = Fraction(0)
    for coeff, mono in terms:
        prod = Fraction(coeff)
        for name, exp in mono:
            prod *= Fraction(assignment[name]) ** exp
        total += prod
    return total


@dataclass(frozen=True)
class Constraint:
    rel: str  # 'le' | 'lt' | 'eq'  (normalised: poly REL 0)
    poly: tuple  # ((coeff_str, ((name, exp), ...)), ...)
    initial: bool
    text: str

    def holds(self, assignment) -> bool:
        v = _eval_poly(self.poly, assignment)
        if self.rel == "le":
            return v <= 0
        if self.rel == "lt":
            return v < 0
        return v == 0

    def variables(self) -> set[str]:
        return {n for _, mono in self.poly for n, _ in mono}


@dataclass(frozen=True)
class Case:
    index: int
    applied: tuple[str, ...]
    trail: tuple[str, ...]
    program: str
    params: tuple[str, ...]
    constraints: tuple[Constraint, ...]
    header: tuple[str, ...]
    witness: dict | None

    def holds(self, assignment) -> bool:
        return all(c.holds(assignment) for c in self.constraints)

    def failing(self, assignment) -> list[str]:
        return [c.text for c in self.constraints if not c.holds(assignment)]

    @property
    def source_applied(self) -> tuple[str, ...]:
        return tuple(s for s in self.applied if s in SOURCE_STRATEGIES)


@dataclass(frozen=True)
class CaseTable:
    family: str
    machine: str
    order: tuple[str, ...]
    params: tuple[str, ...]
    machine_params: tuple[dict, ...]
    cases: tuple[Case, ...]
    source: str
    tree: dict
    counters: tuple[dict, ...] = ()

    def machine_names(self) -> tuple[str, ...]:
        return tuple(p["name"] for p in self.machine_params)

    def holding(self, assignment) -> list[Case]:
        return [c for c in self.cases if c.holds(assignment)]


def _load(path: str) -> CaseTable:
    with open(path) as fh:
        doc = json.load(fh)
    cases = []
    for c in doc["cases"]:
        cons = tuple(
            Constraint(
                k["rel"],
                tuple((t[0], tuple((n, int(e)) for n, e in t[1])) for t in k["poly"]),
                bool(k["initial"]),
                k["text"],
            )
            for k in c["constraints"]
        )
        cases.append(
            Case(
                int(c["index"]),
                tuple(c["applied"]),
                tuple(c["trail"]),
                c["program"],
                tuple(c["params"]),
                cons,
                tuple(c["header"]),
                c["witness"],
            )
        )
    return CaseTable(
        doc["family"],
        doc["machine"],
        tuple(doc["order"]),
        tuple(doc["params"]),
        tuple(doc["machine_params"]),
        tuple(cases),
        doc["source"],
        doc.get("tree", {}),
        tuple(doc.get("counters", ())),
    )


@lru_cache(maxsize=None)
def table(family: str, machine: str = "b200") -> CaseTable:
    """Case table of ``family`` built for machine model ``machine``
    ('b200' = data/b200.machine, 'fermi' = the reference's default model,
    'addition-target' = data/addition.machine)."""
    path = os.path.join(DATA, "cases", "%s.%s.json" % (family, machine))
    if not os.path.exists(path) and machine == "fermi" and family == "addition":
        path = os.path.join(DATA, "cases", "addition.addition-target.json")
    if not os.path.exists(path):
        raise KeyError("no case table for %s on machine %r" % (family, machine))
    return _load(path)


@dataclass(frozen=True)
class Selection:
    """Outcome of evaluating the case discussion at one point."""

    family: str
    machine: str
    case: Case
    assignment: dict
    fallback: bool = False  # no case holds (e.g. a block beyond T_B): most-reduced leaf used

    @property
    def applied(self) -> tuple[str, ...]:
        return self.case.source_applied

    @property
    def index(self) -> int:
        return self.case.index


def select(kind_or_family, params: dict, machine=None) -> Selection:
    """Pick the case whose constraint system holds at params + machine values.

    ``machine``: None / 'live' (device 0's properties through
    pk_query_machine, evaluated on the b200 table), 'fermi' (the reference's
    default machine model, evaluated at its declared limits), or a
    ``MachineValues``.
    """
    family = kind_or_family.family if isinstance(kind_or_family, ProgramKind) else kind_or_family
    mv = machine_mod.resolve(machine)
    tab = table(family, mv.table)
    assignment = {k: Fraction(int(v)) for k, v in params.items() if k in tab.params}
    missing = [p for p in tab.params if p not in assignment]
    if missing:
        raise KeyError("no value supplied for parameter %r" % missing[0])
    for name in tab.machine_names():
        if name not in mv.values:
            raise KeyError("machine model %r needs a value for %r" % (mv.table, name))
        assignment[name] = Fraction(mv.values[name])
    for c in tab.counters:
        # the occupancy counter's warp_slots is a number baked into the table;
        # it must be the device's resident-warp count for the table to apply
        if c.get("measure") == "occupancy":
            built, have = int(c["options"].get("warp_slots", 48)), machine_mod.warp_slots(mv)
            if have is not None and have != built:
                raise ValueError("case table %s.%s assumes %d warp slots per SM; device %s has %d"
                                 % (family, mv.table, built, mv.source, have))
    hold = tab.holding(assignment)
    if len(hold) > 1:  # the leaves partition the box; keep the first (tree order) if not
        hold = hold[:1]
    if hold:
        return Selection(family, mv.table, hold[0], assignment)
    # Outside every leaf (negative parameters, or a thread block the device
    # cannot launch): the program still has a meaning, so run it on the most
    # reduced leaf (the last one of the tree walk) and flag the selection.
    return Selection(family, mv.table, tab.cases[-1], assignment, fallback=True)
