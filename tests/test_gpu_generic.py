"""The generic path on the GPU: programs outside the seven families run
through our own parser and emitted kernel (generic.py, NVRTC for sm_100a),
with no parakern at run time.

* every run the reference interpreter recorded (tests/golden/generic_vectors.json:
  hand-written and random race-free programs, ints, wide ints, binary64 floats
  with specials, mixed lists, bools and objects) gives the reference's arrays
  bit for bit with their Python types, or the reference's exception -- except
  where the reference's unbounded ints leave int64, where the GPU path raises
  OverflowError (the restated interpreter says when: its ``wide`` flag);
* the seven family programs forced through the generic path equal the
  hand-written kernels (and so the oracle) on the golden interp vectors;
* randomised programs and inputs against the restated interpreter.
"""

import json
import math
import os
import random
import struct
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))

import generic_programs  # noqa: E402
from oracle import mfk_interp  # noqa: E402

pytestmark = pytest.mark.gpu

ERRORS = {"IndexError": IndexError, "ZeroDivisionError": ZeroDivisionError, "KeyError": KeyError,
          "TypeError": TypeError, "OverflowError": OverflowError}


@pytest.fixture(scope="module")
def golden():
    with open(os.path.join(HERE, "golden", "generic_vectors.json")) as fh:
        return json.load(fh)


def same(g, w) -> bool:
    if isinstance(w, list):
        return isinstance(g, list) and len(g) == len(w) and all(same(x, y) for x, y in zip(g, w))
    if isinstance(w, float):
        if not isinstance(g, float):
            return False
        return math.isnan(g) if math.isnan(w) else struct.pack("<d", g) == struct.pack("<d", w)
    return type(g) is type(w) and g == w


def _run(text, params, arrays):
    import warnings

    from paper_1801_04348_b200 import run_program

    with warnings.catch_warnings():
        warnings.simplefilter("ignore", RuntimeWarning)
        return run_program(text, dict(params), arrays)


def _check(text, params, arrays, want=None, error=None):
    """One run against the reference's outputs / exception, the restated
    interpreter deciding whether an int left int64 on the way."""
    from paper_1801_04348_b200 import mfk

    # the exceptions any parallel schedule may report: every iteration run on
    # its own by the restated interpreter (the reference stops at the
    # sequentially first one), OverflowError where an int left int64
    stats = {}
    try:
        mfk_interp.run_program(mfk.parse(text), dict(params), json.loads(json.dumps(arrays)), stats=stats,
                               all_iterations=True)
    except (IndexError, ZeroDivisionError, KeyError, TypeError) as exc:  # outside the nest (declarations)
        stats.setdefault("errors", set()).add(type(exc))
    allowed = set(stats.get("errors", ()))
    if error:
        assert ERRORS[error] in allowed or stats.get("wide"), (error, allowed)
    if stats.get("wide"):
        allowed.add(OverflowError)
    try:
        got = _run(text, params, json.loads(json.dumps(arrays)))
    except tuple(ERRORS.values()) as exc:
        assert type(exc) in allowed, (type(exc).__name__, error, str(exc))
        return "raised"
    assert error is None, "expected %s" % error
    assert not stats.get("wide") or want is not None
    assert set(got) == set(want)
    for k in want:
        assert same(got[k], want[k]), (k, got[k][:8] if isinstance(got[k], list) else got[k], want[k][:8])
    return "ok"


def test_golden_runs_match_the_reference(cuda, golden):
    from paper_1801_04348_b200 import last_run

    tally = {"ok": 0, "raised": 0}
    for entry in golden["programs"]:
        for r in entry["runs"]:
            tally[_check(entry["text"], entry["params"], r["inputs"], r.get("outputs"), r.get("error"))] += 1
            assert last_run().family == "generic"
        if entry.get("missing_param"):
            p2 = {k: v for k, v in entry["params"].items() if k != entry["missing_param"]["drop"]}
            with pytest.raises(KeyError):
                _run(entry["text"], p2, None)
    assert tally["ok"] >= 200, tally


def test_value_models_and_mappings_are_exercised(cuda, golden):
    from paper_1801_04348_b200 import generic

    seen = set()
    for entry in golden["programs"]:
        for r in entry["runs"]:
            if "outputs" not in r:
                continue
            try:
                _run(entry["text"], entry["params"], json.loads(json.dumps(r["inputs"])))
            except OverflowError:
                continue
            seen.add((generic.last.mode, generic.last.flat))
    assert {("int", True), ("int", False), ("dyn", True), ("dyn", False)} <= seen


@pytest.mark.parametrize("family", ["reverse", "transpose", "jacobi", "jacobi2d", "matvec", "matmul", "addition"])
def test_family_programs_through_the_generic_path_equal_their_kernels(cuda, family):
    """The emitted kernel and the hand-written leaves agree on the golden
    interp vectors of every family (ints), original programs."""
    from paper_1801_04348_b200 import programs, run_program

    with open(os.path.join(HERE, "golden", "interp_vectors.json")) as fh:
        vecs = [v for v in json.load(fh)["vectors"] if v["family"] == family and v.get("program", "original")
                == "original"][:6]
    assert vecs
    text = programs.source(family)
    for v in vecs:
        inputs = v.get("inputs") or v.get("arrays") or {}
        a = run_program(text, dict(v["params"]), json.loads(json.dumps(inputs)))
        b = run_program(text, dict(v["params"]), json.loads(json.dumps(inputs)), via_generic=True)
        assert set(a) == set(b)
        for k in a:
            assert same(b[k], a[k]), (family, k)


def test_numpy_containers_and_dtypes(cuda):
    text = ("int N;\nint a[N];\nint b[N];\nint c[N];\nmeta_schedule {\n meta_for (int i = 0; i < N; i++)\n"
            "  c[i] = a[i] * 3 - b[(i + 1) % N] / 2;\n}\n")
    N = 1000
    a = np.arange(N, dtype=np.int32) - 500
    b = (np.arange(N, dtype=np.int32) * 7) % 13 - 6
    out = _run(text, {"N": N}, {"a": a, "b": b})
    want = [int(a[i]) * 3 - int(np.trunc(int(b[(i + 1) % N]) / 2)) for i in range(N)]
    assert out["c"].dtype == np.int64 and out["c"].tolist() == want  # c was not supplied: int64 words
    assert out["a"] is not a and out["a"].dtype == np.int32 and (out["a"] == a).all()
    f = _run(text, {"N": N}, {"a": a.astype(np.float64) + 0.25, "b": b})
    assert f["c"].dtype == np.float64
    assert f["c"][0] == (a[0] + 0.25) * 3 - math.copysign(abs(int(b[1])) // 2, int(b[1]))


def test_errors_and_large_grids(cuda):
    text = ("int N;\nint a[N];\nint c[N];\nmeta_schedule {\n meta_for (int i = 0; i < N; i++)\n"
            "  c[i] = a[i] / (i - 7);\n}\n")
    with pytest.raises(ZeroDivisionError):
        _run(text, {"N": 10}, {"a": list(range(10))})
    text2 = ("int N;\nint a[N];\nint c[N];\nmeta_schedule {\n meta_for (int i = 0; i < N; i++)\n"
             "  c[i] = a[i + 1];\n}\n")
    with pytest.raises(IndexError):
        _run(text2, {"N": 10}, {"a": list(range(10))})
    assert _run(text2, {"N": 10}, {"a": list(range(11))})["c"] == list(range(1, 11))  # a longer array is fine
    # a big flat nest: 2^24 iterations over a grid-stride loop
    N = 1 << 24
    text3 = ("int N, B;\nint c[N];\nint d = N / B;\nmeta_schedule {\n meta_for (int i = 0; i < d; i++)\n"
             "  meta_for (int j = 0; j < B; j++)\n   c[i * B + j] = (i * B + j) % 1000 - j;\n}\n")
    out = _run(text3, {"N": N, "B": 64}, {"c": np.zeros(N, dtype=np.int64)})
    idx = np.arange(N, dtype=np.int64)
    assert (out["c"] == idx % 1000 - idx % 64).all()


@pytest.mark.parametrize("seed", range(6))
def test_random_programs_against_the_restated_interpreter(cuda, seed):
    from paper_1801_04348_b200 import mfk

    draws = int(os.environ.get("PK_GENERIC_DRAWS", "24"))
    rng = random.Random(0xC0DE + seed)
    for k in range(draws):
        shape = ["map1d", "map2d", "stencil", "triangle"][(k + seed) % 4]
        text, params = generic_programs.program(rng, shape, safe_div=rng.random() < 0.8,
                                                oob=shape != "stencil" and rng.random() < 0.2)
        style = rng.choice(["int", "wide", "float", "mixed"])
        arrays = generic_programs.inputs(rng, (text, params), style)
        try:
            want = mfk_interp.run_program(mfk.parse(text), dict(params), json.loads(json.dumps(arrays)))
            err = None
        except (IndexError, ZeroDivisionError, KeyError, TypeError) as exc:
            want, err = None, type(exc).__name__
        _check(text, params, arrays, want, err)


def test_run_block_matches_the_reference(cuda, golden):
    """run_block of programs outside the families (generic.run_block): the
    reference's arrays, or its IndexError past the grid."""
    import warnings

    from paper_1801_04348_b200 import last_run, run_block

    n = 0
    for entry in golden["programs"]:
        for b in entry.get("blocks", ()):
            args = (entry["text"], dict(entry["params"]), b["grid_values"], b["context_values"],
                    json.loads(json.dumps(b["inputs"])))
            with warnings.catch_warnings():
                warnings.simplefilter("ignore", RuntimeWarning)
                if "error" in b:
                    with pytest.raises(ERRORS[b["error"]]):
                        run_block(*args)
                else:
                    got = run_block(*args)
                    assert last_run().family == "generic"
                    for k in b["outputs"]:
                        assert same(got[k], b["outputs"][k]), (entry["name"], k)
            n += 1
    assert n >= 100
