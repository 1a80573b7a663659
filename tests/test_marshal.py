"""CPU tests of the value marshalling (paper_1801_04348_b200/marshal.py):
which element type a call runs in, and the host-side word conversions.
No GPU: the kernels are exercised by tests/test_gpu_values.py."""

import json
import os

import numpy as np
import pytest

from paper_1801_04348_b200 import _lib, marshal

HERE = os.path.dirname(os.path.abspath(__file__))
REV = {"N": 8, "s": 1, "B": 4}


@pytest.mark.parametrize("arrays,dtype,objects", [
    ({"a": [1, 2, 3, 4, 5, 6, 7, 8]}, _lib.DTYPE_I32, False),
    ({"a": [0.5] * 8}, _lib.DTYPE_I64, True),  # binary64 floats: object words
    ({"a": [2**40] * 8}, _lib.DTYPE_I64, True),
    ({"a": [True, 1, 2.0, "x"] * 2}, _lib.DTYPE_I64, True),
    ({"a": np.zeros(8)}, _lib.DTYPE_F64, False),
    ({"a": np.zeros(8, np.float32)}, _lib.DTYPE_F32, False),
    ({"a": np.zeros(8, np.int64)}, _lib.DTYPE_I64, False),
    ({"a": np.zeros(8, np.int16)}, _lib.DTYPE_I32, False),
])
def test_permutation_plans(arrays, dtype, objects):
    pl, _ = marshal.plan("reverse", REV, arrays)
    assert (pl.dtype, pl.objects) == (dtype, objects)


def test_arith_plans_pick_exact_types():
    P = {"N": 4, "s": 1, "B": 2}
    small = {"a": [[3] * 4] * 4, "x": [5] * 4}
    assert marshal.plan("matvec", P, small)[0].dtype == _lib.DTYPE_I32
    wide = {"a": [[2**20] * 4] * 4, "x": [2**20] * 4}  # results 2^42: int64
    assert marshal.plan("matvec", P, wide)[0].dtype == _lib.DTYPE_I64
    with pytest.raises(OverflowError):
        marshal.plan("matvec", P, {"a": [[2**40] * 4] * 4, "x": [2**40] * 4})
    assert marshal.plan("matvec", P, {"a": [[0.5] * 4] * 4})[0].dtype == _lib.DTYPE_F64
    assert marshal.plan("matvec", P, {"a": np.ones((4, 4), np.float32)})[0].dtype == _lib.DTYPE_F32
    assert marshal.plan("matvec", P, {"a": np.ones((4, 4), np.float32), "x": np.ones(4)})[0].dtype == _lib.DTYPE_F64
    with pytest.raises(TypeError):
        marshal.plan("matvec", P, {"a": [["x"] * 4] * 4})
    J = {"T": 1, "N": 6, "s": 1, "B": 2}
    assert marshal.plan("jacobi", J, {"a": [0.5] * 12})[0].dtype == _lib.DTYPE_F64  # c_div on Python floats
    assert marshal.plan("jacobi", J, {"a": np.ones(12, np.float32)})[0].dtype == _lib.DTYPE_F64
    assert marshal.plan("jacobi", J, {"a": [2**31] * 12})[0].dtype == _lib.DTYPE_I64
    with pytest.raises(OverflowError):
        marshal.plan("jacobi", J, {"a": [2**62] * 12})


def test_int_bound_is_an_upper_bound_on_the_reference_results():
    """The int32 / int64 decision rests on int_bound: check it dominates the
    reference's own results on the value vectors."""
    with open(os.path.join(HERE, "golden", "value_vectors.json")) as fh:
        vecs = json.load(fh)["vectors"]
    seen = 0
    for v in vecs:
        if v["style"] not in ("i_wide", "i_huge"):
            continue
        srcs = {n: marshal.describe(n, x) for n, x in v["inputs"].items()}
        bound = marshal.int_bound(v["family"], v["params"], srcs)
        for arr in v["outputs"].values():
            flat = arr if not arr or not isinstance(arr[0], list) else [x for r in arr for x in r]
            assert max(abs(x) for x in flat) <= bound
        seen += 1
    assert seen >= 10


def test_object_words_round_trip():
    arrays = {"a": [1.5, -0.0, 2**70, True, "s", None, 3, float("inf")]}
    pl, srcs = marshal.plan("reverse", REV, arrays)
    buf = np.empty(8, np.int64)
    marshal.host_words(pl, srcs["a"], 8, buf)
    back = marshal.finish(pl, srcs["a"], buf, (8,), "list")
    assert all(x is y for x, y in zip(back, arrays["a"]))  # the very objects
    marshal.host_words(pl, None, 8, buf)
    assert marshal.finish(pl, None, buf, (8,), "list") == [0] * 8
    assert all(type(x) is int for x in marshal.finish(pl, None, buf, (8,), "list"))


def test_numpy_words_keep_caller_dtype():
    a = np.arange(8, dtype=np.int16)
    pl, srcs = marshal.plan("reverse", REV, {"a": a})
    buf = np.empty(8, pl.np_dtype)
    marshal.host_words(pl, srcs["a"], 8, buf)
    out = marshal.finish(pl, srcs["a"], buf, (8,), "numpy")
    assert out.dtype == np.int16 and np.array_equal(out, a)
    f = np.array([1.0, -0.0, np.inf, 5e-324] * 2)
    pl, srcs = marshal.plan("reverse", REV, {"a": f})
    buf = np.empty(8, pl.np_dtype)
    marshal.host_words(pl, srcs["a"], 8, buf)
    assert np.array_equal(buf.view(np.uint64), f.view(np.uint64))
