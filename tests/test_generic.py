"""The generic path's front end and its checker, on CPU.

* mfk.parse accepts exactly the texts the reference's dsl.parse accepts and
  finds the same structure (scalars, arrays, bindings, context loops, the
  meta_for nest and its grid / thread roles) -- tests/golden/generic_vectors.json
  records the reference's own verdicts (make_generic.py);
* the pure-Python restatement of the interpreter (oracle/mfk_interp.py) that
  the GPU fuzz tests check against equals the reference interpreter on every
  recorded run (outputs bit for bit, with Python types, or the same exception);
* the emitter produces CUDA text for every recorded program in both value
  models (compiled here with nvcc for a sample; NVRTC compiles them on the GPU).
"""

import json
import math
import os
import struct
import subprocess
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

from oracle import mfk_interp  # noqa: E402
from paper_1801_04348_b200 import generic, mfk  # noqa: E402


@pytest.fixture(scope="module")
def golden():
    with open(os.path.join(HERE, "golden", "generic_vectors.json")) as fh:
        return json.load(fh)


def same(g, w) -> bool:
    """Equal values of equal Python types; floats bit for bit (NaN by NaN)."""
    if isinstance(w, list):
        return isinstance(g, list) and len(g) == len(w) and all(same(x, y) for x, y in zip(g, w))
    if isinstance(w, float):
        if not isinstance(g, float):
            return False
        return math.isnan(g) if math.isnan(w) else struct.pack("<d", g) == struct.pack("<d", w)
    return type(g) is type(w) and g == w


def test_parser_accepts_and_structures_like_the_reference(golden):
    for entry in golden["programs"]:
        p = mfk.parse(entry["text"])
        st = entry["structure"]
        assert p.scalars == st["scalars"], entry["name"]
        assert list(p.arrays) == list(st["arrays"]), entry["name"]
        assert [len(d) for d in p.arrays.values()] == [len(d) for d in st["arrays"].values()], entry["name"]
        assert [b for b, _ in p.bindings] == st["bindings"], entry["name"]
        assert [v for v, _ in p.context] == st["context"], entry["name"]
        assert [m[0] for m in p.meta] == st["meta"], entry["name"]
        assert [m[0] for m in p.grid] == st["grid"], entry["name"]
        assert [m[0] for m in p.thread] == st["thread"], entry["name"]


def test_parser_rejects_what_the_reference_rejects(golden):
    assert len(golden["rejected"]) >= 15
    for entry in golden["rejected"]:
        with pytest.raises(mfk.MfkError):
            mfk.parse(entry["text"])


def test_parser_on_the_family_programs():
    from paper_1801_04348_b200 import programs

    for fam in programs.FAMILIES:
        p = mfk.parse(programs.source(fam))
        assert 2 <= len(p.meta) <= 4 and p.grid and p.thread


def test_oracle_equals_the_reference_interpreter(golden):
    runs = 0
    for entry in golden["programs"]:
        prog = mfk.parse(entry["text"])
        for r in entry["runs"]:
            inputs = json.loads(json.dumps(r["inputs"]))
            if "error" in r:
                with pytest.raises(getattr(__builtins__, r["error"], None) or eval(r["error"])):
                    mfk_interp.run_program(prog, dict(entry["params"]), inputs)
            else:
                got = mfk_interp.run_program(prog, dict(entry["params"]), inputs)
                assert set(got) == set(r["outputs"]), entry["name"]
                for k in got:
                    assert same(got[k], r["outputs"][k]), (entry["name"], r["style"], k)
            runs += 1
        if entry.get("missing_param"):
            p2 = {k: v for k, v in entry["params"].items() if k != entry["missing_param"]["drop"]}
            with pytest.raises(KeyError):
                mfk_interp.run_program(prog, p2)
    assert runs >= 250


def test_emitter_covers_every_golden_program(golden):
    for entry in golden["programs"]:
        prog = mfk.parse(entry["text"])
        names = list(prog.arrays)
        ids = {n: k for k, n in enumerate(names)}
        ranks = {n: len(d) for n, d in prog.arrays.items()}
        env = sorted(set(entry["params"]) | {b for b, _ in prog.bindings}) + [v for v, _ in prog.context]
        for mode in ("int", "dyn"):
            for flat in (True, False):
                src = generic._Emitter(prog, mode, env, ids, ranks, flat).kernel()
                assert 'extern "C" __global__' in src and "pk_generic(" in src


@pytest.mark.parametrize("name", ["branch", "pingpong2d", "grid3"])
def test_emitted_text_compiles_for_sm100a(golden, tmp_path, name):
    entry = next(e for e in golden["programs"] if e["name"] == name)
    prog = mfk.parse(entry["text"])
    names = list(prog.arrays)
    env = sorted(set(entry["params"]) | {b for b, _ in prog.bindings}) + [v for v, _ in prog.context]
    for mode in ("int", "dyn"):
        src = generic._Emitter(prog, mode, env, {n: k for k, n in enumerate(names)},
                               {n: len(d) for n, d in prog.arrays.items()}, False).kernel()
        f = tmp_path / ("%s_%s.cu" % (name, mode))
        f.write_text(src)
        r = subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-c", str(f), "-o",
                            str(tmp_path / "k.o")], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr[-2000:]


def test_host_eval_is_c_division():
    env = {"a": -7, "b": 2}
    e = mfk.parse("int a, b;\nint x = a / b;\nint y = a % b;\nint c[1];\n"
                  "meta_schedule { meta_for (int i = 0; i < 1; i++) c[i] = x; }\n")
    vals = {n: generic.host_eval(v, env) for n, v in e.bindings}
    assert vals == {"x": -3, "y": -1}
    with pytest.raises(ZeroDivisionError):
        generic.host_eval(("bin", "/", ("num", 1), ("num", 0)), {})
    with pytest.raises(KeyError):
        generic.host_eval(("name", "missing"), {})


def test_oracle_run_block_equals_the_reference(golden):
    n = 0
    for entry in golden["programs"]:
        prog = mfk.parse(entry["text"])
        for b in entry.get("blocks", ()):
            args = (prog, dict(entry["params"]), b["grid_values"], b["context_values"],
                    json.loads(json.dumps(b["inputs"])))
            if "error" in b:
                with pytest.raises(eval(b["error"])):
                    mfk_interp.run_block(*args)
            else:
                got = mfk_interp.run_block(*args)
                for k in b["outputs"]:
                    assert same(got[k], b["outputs"][k]), (entry["name"], k)
            n += 1
    assert n >= 100
