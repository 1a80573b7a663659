"""run_block on the GPU (interp.run_block -> the emitted leaf with its grid
loops pinned, one block) against the reference's own run_block
(tests/golden/run_block_vectors.json, made by tests/golden/make_run_block.py
from parakern.interp.run_block, interp.py:228-249): bit-exact at every grid
point of every family, original and caching-off programs."""

import json
import os

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _vectors():
    with open(os.path.join(HERE, "golden", "run_block_vectors.json")) as fh:
        return json.load(fh)["vectors"]


def test_run_block_matches_reference(cuda):
    from paper_1801_04348_b200 import programs, run_block

    n = 0
    for v in _vectors():
        text = programs.source(v["family"]) if v["variant"] == "original" else v["program"]
        got = run_block(text, v["params"], v["grid_values"], v["context_values"], arrays=v["inputs"])
        for name, want in v["outputs"].items():
            assert got[name] == want, (v["family"], v["variant"], v["grid_values"], v["context_values"], name)
        n += 1
    assert n >= 70


def test_run_block_errors(cuda):
    from paper_1801_04348_b200 import programs, run_block

    text = programs.source("jacobi")
    P = {"T": 2, "N": 26, "s": 2, "B": 4}
    with pytest.raises(KeyError):  # context variable t not supplied
        run_block(text, P, {"i": 0})
    with pytest.raises(IndexError):  # grid value outside the meta_for range
        run_block(text, P, {"i": 3}, {"t": 0})
    with pytest.raises(NotImplementedError):
        run_block(text, P, {"i": 0}, {"t": 0}, tracer=lambda *a: None)


def test_caching_off_programs_run_on_the_direct_kernels(cuda, oracle_mod):
    """The original programs with caching-off alone (strategies.apply_source,
    not a case-tree leaf) are recognised and run on the direct kernels, with
    the original program's results."""
    import numpy as np

    from paper_1801_04348_b200 import last_run, programs, run_program

    texts = {}
    for v in _vectors():
        if v["variant"] == "caching-off":
            texts.setdefault(v["family"], (v["program"], v["params"]))
    rng = np.random.default_rng(3)
    for family, (text, params) in sorted(texts.items()):
        shapes = programs.array_shapes(programs.original(family), params)
        inputs = {k: rng.integers(-1000, 1000, size=s).astype(np.int32) for k, s in shapes.items()}
        want = oracle_mod.run(family, params, inputs)
        got = run_program(text, params, inputs)
        assert last_run().applied == ("caching-off",)
        for name in want:
            assert np.array_equal(np.asarray(got[name]).reshape(-1), np.asarray(want[name]).reshape(-1)), family
