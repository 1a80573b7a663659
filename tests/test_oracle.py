"""The CPU oracle (oracle/pk_oracle.c) pinned against the reference.

* golden vectors produced by the reference interpreter itself
  (tests/golden/make_golden.py -> parakern.interp.run_program, interp.py:215);
* the hand-computed vectors of the reference's own tests
  (pkg/tests/test_interp.py:10-88).
"""

import numpy as np
import pytest


def _as_np(v, floats):
    return np.asarray(v, dtype=np.float64 if floats else np.int64)


def test_c_division_truncates(oracle_mod):
    # pkg/tests/test_interp.py:10-18 -- the oracle's Jacobi uses C '/'
    out = oracle_mod.run("jacobi", {"T": 1, "N": 3, "s": 1, "B": 1}, {"a": [0, 0, 0, -7, 0, 0]})
    assert out["a"][1] == -2  # (-7 + 0 + 0) / 3 truncates toward zero, not -3


def test_jacobi_one_sweep_by_hand(oracle_mod):
    # pkg/tests/test_interp.py:43-53
    seed = [0, 0, 0, 0, 9, 3, 6, 12]
    out = oracle_mod.run("jacobi", {"N": 4, "s": 1, "B": 2, "T": 1}, {"a": seed})
    assert out["a"].tolist() == [0, (9 + 3 + 6) // 3, (3 + 6 + 12) // 3, 0, 9, 3, 6, 12]


def test_jacobi_odd_sweep_by_hand(oracle_mod):
    # pkg/tests/test_interp.py:56-66
    seed = [9, 3, 6, 12, 0, 0, 0, 0]
    out = oracle_mod.run("jacobi", {"N": 4, "s": 1, "B": 2, "T": 2}, {"a": seed})
    assert out["a"][5] == (9 + 0 + 0) // 3
    assert out["a"][6] == (0 + 0 + 12) // 3


def test_transpose_by_hand(oracle_mod):
    # pkg/tests/test_interp.py:69-76
    out = oracle_mod.run("transpose", {"N": 2, "s": 1, "B0": 1, "B1": 1}, {"a": [[1, 2], [3, 4]]})
    assert out["c"].tolist() == [1, 3, 2, 4]


def test_addition_by_hand(oracle_mod):
    # pkg/tests/test_interp.py:79-88
    out = oracle_mod.run("addition", {"N": 2, "B0": 1, "B1": 1}, {"a": [1, 2, 3, 4], "b": [10, 20, 30, 40]})
    assert out["c"].tolist() == [11, 22, 33, 44]


def test_oracle_matches_reference_interpreter(golden, oracle_mod):
    checked = 0
    for v in golden:
        if v.get("error"):
            with pytest.raises(ZeroDivisionError):
                oracle_mod.run(v["family"], v["params"], {})
            continue
        if v.get("error", "missing") is None:
            continue
        params = dict(v["params"])
        merged = False
        if v["program"] != "original":
            if v["family"] == "addition":
                merged = "granularity" in v["applied"]
            else:
                params.setdefault("s", 1)
        floats = v["floats"]
        inputs = {k: _as_np(x, floats) for k, x in v["inputs"].items()}
        got = oracle_mod.run(v["family"], params, inputs, merged=merged)
        for name, want in v["outputs"].items():
            w = _as_np(want, floats)
            g = np.asarray(got[name]).reshape(w.shape)
            if floats:
                # binary64, interpreter order, no contraction: bit-exact
                assert np.array_equal(g.astype(np.float64), w), (v["family"], name, v["params"])
            else:
                assert np.array_equal(g.astype(np.int64), w), (v["family"], name, v["params"])
        checked += 1
    assert checked >= 100
