"""Case-tree evaluation (paper_1801_04348_b200/cases.py) against the
reference engine's own ConstraintSystem.holds (algebra.py:621-622), and the
case splits the reference's tests pin (pkg/tests/test_engine.py:23-85)."""

import json
import os

import pytest

from paper_1801_04348_b200 import cases, machine, programs

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_selection_matches_reference_holds():
    with open(os.path.join(GOLDEN, "case_selection.json")) as fh:
        records = json.load(fh)["records"]
    for r in records:
        tab = cases.table(r["family"], r["machine"])
        assignment = {**r["params"], **r["machine_values"]}
        got = [c.index for c in tab.cases if c.holds(assignment)]
        assert got == r["holding"], r


@pytest.mark.parametrize("family,count", [("jacobi", 7), ("transpose", 4), ("addition", 2),
                                          ("matmul", 4), ("reverse", 4), ("matvec", 3), ("jacobi2d", 4)])
def test_case_counts(family, count):
    # jacobi 7 / transpose 4 / addition 2: pkg/tests/test_engine.py:23-85;
    # the SURVEY App. A programs: 4 / 4 / 3 / 4 on the Fermi model
    assert len(cases.table(family, "fermi").cases) == count


def test_jacobi_fermi_headers_match_reference_split():
    # pkg/tests/test_acceptance.py c01 / test_engine.py: case 1 keeps cache + s,
    # case 6 is granularity + caching-off below 2*B + 2 words
    tab = cases.table("jacobi", "fermi")
    assert tab.cases[0].header == ("2*s*B + 2 <= Z_B", "10 <= R_B")
    assert tab.cases[5].source_applied == ("granularity", "caching-off")
    assert tab.cases[5].header == ("Z_B < 2*B + 2", "7 <= R_B")


def test_fermi_selects_case1_for_paper_matmul_shapes():
    # all 7 Table-1 shapes x s in {2,4} x n in {1024, 2048}
    # select case 1 (no strategies) on the reference's default machine
    shapes = [(2, 4), (4, 4), (8, 4), (16, 8), (32, 8), (8, 16), (16, 16)]  # (ub1, B0)
    for ub1, B0 in shapes:
        for s in (2, 4):
            for n in (1024, 2048):
                sel = cases.select("matmul", {"n": n, "B0": B0, "ub1": ub1, "s": s}, machine.fermi())
                assert sel.index == 1 and sel.applied == ()


def test_live_values_change_the_selection():
    # Z_B = 58112 (opt-in) vs 12288 (static) flips mat-vec at N = 16384
    opt = machine.nominal("optin")
    static = machine.nominal("static")
    p = {"N": 16384, "s": 1, "B": 256}
    assert cases.select("matvec", p, opt).applied == ()
    assert cases.select("matvec", p, static).applied == ("granularity", "caching-off")
    # reversal: s*B words staged if they fit, else granularity (B fits), else caching-off
    assert cases.select("reverse", {"N": 1 << 30, "s": 64, "B": 1024}, opt).applied == ("granularity",)
    assert cases.select("reverse", {"N": 1 << 30, "s": 16, "B": 256}, opt).applied == ()


def test_out_of_box_point_falls_back_to_most_reduced_leaf():
    sel = cases.select("transpose", {"N": 64, "s": 1, "B0": 64, "B1": 64}, machine.nominal())
    assert sel.fallback and sel.applied == ("granularity", "caching-off")


def test_missing_parameter_is_keyerror():
    with pytest.raises(KeyError):
        cases.select("jacobi", {"T": 1, "N": 10, "s": 1}, machine.nominal())


def test_every_table_case_program_is_recognised():
    for path in programs.case_tables():
        doc = json.load(open(path))
        assert programs.identify(doc["source"]).is_original
        for c in doc["cases"]:
            kind = programs.identify(c["program"])
            assert kind.family == doc["family"]
            assert kind.applied == tuple(s for s in c["applied"] if s in programs.SOURCE_STRATEGIES)


def test_machine_file_text_parses_with_reference_syntax():
    import configparser

    text = machine.machine_file_text(machine.nominal())
    cp = configparser.ConfigParser(interpolation=None)
    cp.optionxform = str  # as parse_machine does (machine.py:112)
    cp.read_string(text)
    assert cp["param.Z_B"]["range"] == "0 58112"
    assert cp["counter.threads"]["bound"] == "T_B"


# ---- occupancy model (data/b200-occ.machine) -----------------

OCC_FAMILIES = ("addition", "jacobi", "jacobi2d", "matmul", "matvec", "reverse", "transpose")


def test_occupancy_tables_carry_the_counter():
    for fam in OCC_FAMILIES:
        tab = cases.table(fam, "b200-occ")
        assert {"R_F", "O"} <= set(tab.machine_names())
        (occ,) = [c for c in tab.counters if c["measure"] == "occupancy"]
        assert occ["bound"] == "O" and occ["options"]["register_file"] == "R_F"
        assert int(occ["options"]["warp_slots"]) == 64  # 2048 threads / 32 per SM on sm_100
        # the counter only restricts: same leaves (applied tuples) as the b200 table
        assert [c.applied for c in tab.cases] == [c.applied for c in cases.table(fam, "b200").cases]
        for c in tab.cases:
            assert any("R_F" in k.text and "O" in k.text for k in c.constraints)


def test_occupancy_constraint_is_the_reference_ratio():
    # counters.py:512-524: R_F / (threads * regs * warp_slots) <= O, regs = the
    # case program's peak live registers (10 for the original 1-D Jacobi)
    from fractions import Fraction

    mv0 = machine.nominal(occupancy=1)
    for B in (64, 96, 102, 103, 128, 256, 1024):
        for O in (Fraction(1), Fraction(1, 2), Fraction(1, 5)):
            mv = machine.MachineValues("b200-occ", dict(mv0.values, O=O), "user", mv0.props)
            sel = cases.select("jacobi", {"T": 4, "N": 4098, "s": 2, "B": B}, mv)
            ratio = Fraction(65536, B * 10 * 64)
            assert (not sel.fallback and sel.index == 1) == (ratio <= O), (B, O)


def test_occupancy_selection_refines_b200():
    mv_occ, mv = machine.nominal(occupancy=1), machine.nominal()
    P = {"n": 8192, "B0": 128, "ub1": 8, "s": 16}
    assert cases.select("matmul", P, mv_occ).index == cases.select("matmul", P, mv).index == 1
    # a 64-thread reversal block cannot reach the ratio on a 64K register file
    sel = cases.select("reverse", {"N": 1 << 20, "s": 16, "B": 64}, mv_occ)
    assert sel.fallback


def test_occupancy_target_range_and_warp_slots_checked():
    with pytest.raises(ValueError):
        machine.nominal(occupancy=2)
    mv = machine.nominal(occupancy=1)
    odd = machine.MachineValues("b200-occ", mv.values, "user", dict(mv.props, max_threads_per_sm=1536))
    with pytest.raises(ValueError, match="warp slots"):
        cases.select("jacobi", {"T": 4, "N": 4098, "s": 2, "B": 256}, odd)
    with pytest.raises(KeyError):
        cases.select("jacobi", {"T": 4, "N": 4098, "s": 2, "B": 256},
                     machine.MachineValues("b200-occ", machine.nominal().values, "user"))


def test_surviving_leaves_match_reference_consistency_checker():
    """a7: the leaves that can hold once the machine is fixed -- our
    restatement of check_consistency against the reference's own verdicts
    (tests/golden/survival.json, make_survival.py)."""
    import json
    import os
    from fractions import Fraction

    from paper_1801_04348_b200 import cases, machine

    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "survival.json")
    with open(path) as fh:
        tables = json.load(fh)["tables"]
    models = {"b200": machine.nominal(), "b200-static": machine.nominal(smem="static"),
              "b200-occ": machine.nominal(occupancy=Fraction(1, 2)), "fermi": machine.fermi()}
    checked = 0
    for t in tables:
        got = cases.surviving(t["family"], models[t["model"]], all_leaves=True)
        assert [(s.case.index, s.status) for s in got] == [(v["case"], v["status"]) for v in t["verdicts"]], \
            (t["family"], t["model"])
        for s in got:  # a witness really satisfies the leaf at the fixed machine values
            if s.status == "consistent":
                point = dict(s.witness, **{k: Fraction(v) for k, v in t["values"].items()})
                assert s.case.holds(point)
        checked += 1
    assert checked >= 28
