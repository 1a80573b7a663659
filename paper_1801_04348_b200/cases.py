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


def select(kind_or_family, params: dict, machine=None, among=None) -> Selection:
    """Pick the case whose constraint system holds at params + machine values.

    ``machine``: None / 'live' (device 0's properties through
    pk_query_machine, evaluated on the b200 table), 'fermi' (the reference's
    default machine model, evaluated at its declared limits), or a
    ``MachineValues``.  ``among``: evaluate only these case indices (the
    leaves :func:`surviving` left at this machine -- the others cannot hold).
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
    hold = tab.holding(assignment) if among is None else \
        [c for c in tab.cases if c.index in among and c.holds(assignment)]
    if len(hold) > 1:  # the leaves partition the box; keep the first (tree order) if not
        hold = hold[:1]
    if hold:
        return Selection(family, mv.table, hold[0], assignment)
    # Outside every leaf (negative parameters, or a thread block the device
    # cannot launch): the program still has a meaning, so run it on the most
    # reduced leaf (the last one of the tree walk) and flag the selection.
    return Selection(family, mv.table, tab.cases[-1], assignment, fallback=True)


# ---------------------------------------------------------------------------
# Survival at the live machine (engine.py:514-528 `_machine_feasible`,
# algebra.py:722-911 `check_consistency`): which leaves can hold at all once
# the machine parameters are fixed to the device's values -- is the leaf's
# system satisfiable for some program / data parameters inside the table's
# box?  The reference asks the mirror question (program fixed, machine free);
# the decision procedure is the same: search-free interval refutation
# (algebra.py:668-714 `refute_by_intervals`), then heuristic corner points,
# seeded random probes and, for small boxes, exhaustive enumeration, every
# candidate checked exactly.


def _poly_of(terms) -> dict:
    out: dict = {}
    for coeff, mono in terms:
        key = tuple(sorted(mono))
        out[key] = out.get(key, Fraction(0)) + Fraction(coeff)
    return {k: v for k, v in out.items() if v != 0}


def _poly_mul(p: dict, q: dict) -> dict:
    out: dict = {}
    for m1, c1 in p.items():
        for m2, c2 in q.items():
            exps = dict(m1)
            for n, e in m2:
                exps[n] = exps.get(n, 0) + e
            key = tuple(sorted(exps.items()))
            out[key] = out.get(key, Fraction(0)) + c1 * c2
    return {k: v for k, v in out.items() if v != 0}


def _poly_add(p: dict, q: dict) -> dict:
    out = dict(p)
    for m, c in q.items():
        out[m] = out.get(m, Fraction(0)) + c
    return {k: v for k, v in out.items() if v != 0}


def _poly_subs(p: dict, sub: dict) -> dict:
    """Substitute polynomials (dicts) for variables (algebra.py:171-181)."""
    out: dict = {}
    for mono, coeff in p.items():
        term = {(): coeff}
        for n, e in mono:
            base = sub.get(n, {((n, 1),): Fraction(1)})
            for _ in range(e):
                term = _poly_mul(term, base)
        out = _poly_add(out, term)
    return out


def _mono_bounds(p: dict, box: dict):
    """Monomial-wise interval arithmetic over a nonnegative box (algebra.py:310-322);
    hi None = unbounded."""
    lo_t, hi_t = Fraction(0), Fraction(0)
    for mono, coeff in p.items():
        plo, phi = Fraction(1), Fraction(1)
        for n, e in mono:
            vlo, vhi = box.get(n, (0, None))
            plo *= Fraction(vlo) ** e
            phi = None if (phi is None or vhi is None) else phi * Fraction(vhi) ** e
        if coeff >= 0:
            lo_t += coeff * plo
            hi_t = None if (hi_t is None or phi is None) else hi_t + coeff * phi
        else:
            hi_t = None if hi_t is None else hi_t + coeff * plo
            lo_t = lo_t + coeff * phi if phi is not None else Fraction(-10**30)
    return lo_t, hi_t


def _bounds(p: dict, box: dict):
    """Range of p over the box: the tighter of the direct and the floor-shifted
    monomial bounds (algebra.py:278-307)."""
    dlo, dhi = _mono_bounds(p, box)
    names = {n for mono in p for n, _ in mono}
    shift, sbox = {}, {}
    for n in names:
        lo, hi = box.get(n, (0, None))
        if lo > 0:
            shift[n] = {((n, 1),): Fraction(1), (): Fraction(lo)}
            sbox[n] = (0, None if hi is None else hi - lo)
        else:
            sbox[n] = (lo, hi)
    if not shift:
        return dlo, dhi
    tlo, thi = _mono_bounds(_poly_subs(p, shift), sbox)
    his = [h for h in (dhi, thi) if h is not None]
    return max(dlo, tlo), (min(his) if his else None)


def _eval(p: dict, point: dict) -> Fraction:
    total = Fraction(0)
    for mono, coeff in p.items():
        prod = coeff
        for n, e in mono:
            prod *= point[n] ** e
        total += prod
    return total


def _rel_holds(v: Fraction, rel: str) -> bool:
    return v <= 0 if rel == "le" else v < 0 if rel == "lt" else v == 0


@dataclass(frozen=True)
class Survival:
    case: Case
    status: str  # consistent | inconsistent | unknown
    witness: dict | None = None
    reason: str | None = None


def _consistent(system: list, box: dict, budget: int = 200_000, seed: int = 0x5EED):
    """check_consistency restated (algebra.py:722-911) without solved
    variables: every variable of ``system`` (poly dict, rel) ranges over the
    integers of ``box``."""
    import itertools
    import random

    for p, rel in system:  # single-constraint ranges
        lo, hi = _bounds(p, box)
        if (rel == "le" and lo > 0) or (rel == "lt" and lo >= 0) or \
                (rel == "eq" and (lo > 0 or (hi is not None and hi < 0))):
            return "inconsistent", None, "interval-contradiction"
    ineq = [(p, rel) for p, rel in system if rel != "eq"]
    for (p, r1), (q, r2) in itertools.combinations(ineq, 2):  # pairwise sums
        pv = {n for m in p for n, _ in m}
        qv = {n for m in q for n, _ in m}
        if not (pv & qv):
            continue
        lo, _ = _bounds(_poly_add(p, q), box)
        if ((r1 == "lt" or r2 == "lt") and lo >= 0) or lo > 0:
            return "inconsistent", None, "pairwise-contradiction"
    names = sorted({n for p, _ in system for m in p for n, _ in m})

    def holds(point):
        return all(_rel_holds(_eval(p, point), rel) for p, rel in system)

    if not names:
        return ("consistent", {}, None) if holds({}) else ("inconsistent", None, "exhausted-box")
    cands = []
    for n in names:
        lo, hi = box[n]
        c = {lo, lo + 1, lo + 2, lo + 4, lo + 8, (lo + hi) // 2, hi - 1, hi}
        cands.append(sorted(v for v in c if lo <= v <= hi))
    total = 1
    for c in cands:
        total *= len(c)
    if total <= max(budget // 4, 4096):
        for values in itertools.product(*cands):
            pt = {n: Fraction(v) for n, v in zip(names, values)}
            if holds(pt):
                return "consistent", pt, None
    else:
        rng0 = random.Random(seed ^ 0xC0FFEE)
        for _ in range(4096):
            pt = {n: Fraction(c[rng0.randrange(len(c))]) for n, c in zip(names, cands)}
            if holds(pt):
                return "consistent", pt, None
    rng = random.Random(seed)
    for _ in range(max(budget // 8, 1024)):
        pt = {}
        for n in names:
            lo, hi = box[n]
            if hi - lo > 64 and rng.random() < 0.5:
                pt[n] = Fraction(min(hi, lo + int((hi - lo) ** rng.random())))
            else:
                pt[n] = Fraction(rng.randint(lo, hi))
        if holds(pt):
            return "consistent", pt, None
    size = 1
    for n in names:
        size *= box[n][1] - box[n][0] + 1
        if size > budget:
            return "unknown", None, "budget"
    for values in itertools.product(*[range(box[n][0], box[n][1] + 1) for n in names]):
        pt = {n: Fraction(v) for n, v in zip(names, values)}
        if holds(pt):
            return "consistent", pt, None
    return "inconsistent", None, "exhausted-box"


def _table_box(family: str, table_name: str) -> dict:
    path = os.path.join(DATA, "cases", "%s.%s.json" % (family, table_name))
    if not os.path.exists(path):
        path = os.path.join(DATA, "cases", "%s.%s.json" % (family, table(family, table_name).machine))
    with open(path) as fh:
        box = json.load(fh).get("box", {})
    return {k: (int(v[0]), int(v[1])) for k, v in box.items()}


@lru_cache(maxsize=None)
def _surviving(family: str, table_name: str, values: tuple, budget: int) -> tuple:
    tab = table(family, table_name)
    fixed = {k: {(): Fraction(v)} for k, v in values}
    box = {k: v for k, v in _table_box(family, table_name).items() if k not in fixed}
    out = []
    for case in tab.cases:
        system = [(_poly_subs(_poly_of(c.poly), fixed), c.rel) for c in case.constraints]
        status, witness, reason = _consistent(system, box, budget=budget)
        out.append(Survival(case, status, witness, reason))
    return tuple(out)


def surviving(family: str, machine=None, *, all_leaves: bool = False, budget: int = 200_000,
              maybe: bool = False):
    """The leaves of ``family``'s case discussion that can hold at the
    machine's values (default: the live device) for some program / data
    parameters in the table's box.  ``all_leaves=True`` returns every leaf's
    :class:`Survival` verdict instead of the surviving cases only;
    ``maybe=True`` also keeps leaves the search could not decide ('unknown')
    -- what a pruner may drop is only what is proven dead."""
    mv = machine_mod.resolve(machine)
    tab = table(family, mv.table)
    values = tuple(sorted((n, Fraction(mv.values[n])) for n in tab.machine_names()))
    res = _surviving(family, mv.table, values, budget)
    if all_leaves:
        return list(res)
    keep = ("consistent", "unknown") if maybe else ("consistent",)
    return [s.case for s in res if s.status in keep]
