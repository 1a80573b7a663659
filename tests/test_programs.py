"""Program identity and parameter handling (paper_1801_04348_b200/programs.py)."""

import pytest

from paper_1801_04348_b200 import _lib, binding, programs


def test_normalize_ignores_comments_and_layout():
    a = programs.source("reverse")
    b = "// a comment\n" + a.replace("    ", "\t").replace(" = ", "=") + "\n/* trailing */"
    assert programs.normalize(a) == programs.normalize(b)
    assert programs.identify(b).family == "reverse"


def test_unknown_program_is_not_implemented():
    with pytest.raises(NotImplementedError):
        programs.identify("int N; int a[N]; meta_schedule { meta_for (int i = 0; i < N; i++) { a[i] = i; } }")


@pytest.mark.parametrize("family", sorted(programs.FAMILIES))
def test_original_programs_identified(family):
    kind = programs.identify(programs.source(family))
    assert kind.family == family and kind.is_original
    assert kind.params == programs.FAMILIES[family].params


def test_missing_parameter_keyerror_names_first_declared():
    kind = programs.original("jacobi")
    with pytest.raises(KeyError, match="'s'"):
        programs.effective_params(kind, {"T": 1, "N": 4, "B": 2})


def test_granularity_program_gets_s_equal_one():
    from paper_1801_04348_b200 import cases

    case = [c for c in cases.table("jacobi", "fermi").cases if c.source_applied == ("granularity",)][0]
    kind = programs.identify(case.program)
    assert kind.applied == ("granularity",)
    P = programs.effective_params(kind, {"T": 2, "N": 10, "B": 4})
    assert P["s"] == 1


def test_array_shapes_follow_declarations():
    assert programs.array_shapes(programs.original("jacobi2d"), {"T": 1, "N": 5, "s": 1, "B0": 1, "B1": 1}) == {"a": (10, 5)}
    assert programs.array_shapes(programs.original("transpose"), {"N": 3, "s": 1, "B0": 1, "B1": 1}) == {"a": (3, 3), "c": (9,)}


def test_binding_variants():
    kind = programs.original("reverse")
    P = {"N": 64, "s": 4, "B": 8}
    L = binding.make_launch(kind, P, ())
    assert L.variant == _lib.VARIANT_STAGED and L.flags == 0
    L = binding.make_launch(kind, P, ("granularity",))
    assert L.variant == _lib.VARIANT_STAGED and L.flags & _lib.FLAG_GRANULARITY
    L = binding.make_launch(kind, P, ("granularity", "caching-off"))
    assert L.variant == _lib.VARIANT_DIRECT
    # merged addition text -> PK_FLAG_MERGED; original addition never merges
    from paper_1801_04348_b200 import cases

    merged_text = [c for c in cases.table("addition", "fermi").cases if c.source_applied][0].program
    mk = programs.identify(merged_text)
    L = binding.make_launch(mk, {"N": 8, "B0": 2, "B1": 2}, mk.applied)
    assert L.flags & _lib.FLAG_MERGED
    L = binding.make_launch(programs.original("addition"), {"N": 8, "B0": 2, "B1": 2}, ("granularity",))
    assert not (L.flags & _lib.FLAG_MERGED)


def test_alpha_renamed_programs_are_recognised():
    """A consistent renaming of identifiers is the same program (the caller's
    names map onto the family's); an inconsistent one is not."""
    import re

    import pytest

    from paper_1801_04348_b200 import programs

    for family in programs.FAMILIES:
        text = programs.source(family)
        names = programs.alpha(programs.normalize(text))[1]
        renamed = text
        for i, n in enumerate(names):
            renamed = re.sub(r"\b%s\b" % n, "zz%d_%s" % (i, n), renamed)
        kind = programs.identify(renamed)
        assert kind.family == family and kind.is_original
        assert dict(kind.rename) == {"zz%d_%s" % (i, n): n for i, n in enumerate(names)}
    broken = programs.source("reverse").replace("c[N - 1 - p]", "a[N - 1 - p]")  # writes a, not c
    with pytest.raises(NotImplementedError):
        programs.identify(broken)
