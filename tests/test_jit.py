"""Emitted-kernel path (paper_1801_04348_b200/jit.py): the reference's own
CUDA text for a leaf, compiled at load time with NVRTC.

CPU: the C-semantics expression evaluator and launch geometry.  GPU: every
shipped emitted leaf (the seven families and two programs outside them,
original and caching-off) against the reference interpreter's vectors."""

import json
import os

import numpy as np
import pytest

from paper_1801_04348_b200 import jit

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "emitted_leaves.json")


def _entries():
    with open(GOLDEN) as fh:
        return json.load(fh)["entries"]


def test_ceval_truncates_like_c():
    assert jit.ceval("(N - 2) / (s * B)", {"N": 26, "s": 2, "B": 8}) == 1
    assert jit.ceval("-7 / 2", {}) == -3
    assert jit.ceval("-7 % 2", {}) == -1
    assert jit.ceval("2 * N * N", {"N": 5}) == 50
    with pytest.raises(ZeroDivisionError):
        jit.ceval("N / s", {"N": 4, "s": 0})
    with pytest.raises(KeyError):
        jit.ceval("N + q", {"N": 1})


def test_leaves_load_and_describe_launches():
    entries = _entries()
    assert {e["program"] for e in entries} >= {"saxpy", "rowsmooth", "jacobi", "matmul"}
    for e in entries:
        leaf = jit.Leaf.from_json(e["leaf"])
        assert "__global__ void " + leaf.kernel_name in leaf.source
        for v in e["vectors"]:
            shapes = jit.array_shapes(leaf, v["params"])
            for name, data in v["inputs"].items():
                n = len(data) * (len(data[0]) if data and isinstance(data[0], list) else 1)
                assert n == int(np.prod(shapes[name]))


@pytest.mark.gpu
def test_emitted_leaves_match_reference_on_gpu(cuda):
    checked = 0
    for e in _entries():
        leaf = jit.Leaf.from_json(e["leaf"])
        for v in e["vectors"]:
            got = jit.run_program_jit(leaf, v["params"], v["inputs"])
            for name, want in v["outputs"].items():
                assert got[name] == want, (e["program"], e["variant"], v["params"], name)
            checked += 1
    assert checked >= 20


def test_block_leaf_pins_every_grid_loop():
    """run_block's kernel: each packaged leaf's grid meta_for loops become a
    single iteration at a kernel argument (no GPU needed)."""
    import re

    from paper_1801_04348_b200 import jit

    for fam in ("addition", "jacobi", "jacobi2d", "matmul", "matvec", "reverse", "transpose"):
        for variant in ("original", "caching-off"):
            if fam == "addition" and variant == "caching-off":
                continue
            leaf = jit.packaged_leaf(fam, variant)
            b = jit.block_leaf(leaf)
            assert "PK_GRID_STRIDE)" not in re.sub(r"#.*", "", b.source.split("__global__")[1])
            for var, _ in leaf.grid:
                assert "int pk_rb_%s" % var in b.source
                assert ("pk_rb_%s" % var, "int") in b.args


@pytest.mark.gpu
def test_emitted_path_refuses_short_and_wide_arrays(cuda):
    """The emitted leaves have no bounds guards: run_program_jit raises
    IndexError for an array shorter than declared (interp.py:209-212) and
    OverflowError for values outside int32, instead of running past the
    buffer or wrapping; undeclared arrays come back as copies."""
    e = next(x for x in _entries() if x["program"] == "saxpy" and x["variant"] == "original")
    leaf = jit.Leaf.from_json(e["leaf"])
    v = e["vectors"][0]
    short = {k: (d[:-1] if not (d and isinstance(d[0], list)) else d[:-1]) for k, d in v["inputs"].items()}
    with pytest.raises(IndexError):
        jit.run_program_jit(leaf, v["params"], short)
    wide = {k: [[2**40] * len(d[0])] * len(d) if d and isinstance(d[0], list) else [2**40] * len(d)
            for k, d in v["inputs"].items()}
    with pytest.raises(OverflowError):
        jit.run_program_jit(leaf, v["params"], wide)
    got = jit.run_program_jit(leaf, v["params"], dict(v["inputs"], extra=[7]))
    assert got["extra"] == [7]
