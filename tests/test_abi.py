"""The C ABI (include/pk.h): libpk.so loads on a CPU-only host, exports every
declared entry point, and the ctypes mirrors match the C layouts."""

import ctypes
import os
import re
import subprocess

import pytest

from paper_1801_04348_b200 import _lib

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "pk.h")


def _declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char \*)\s*(pk_[a-z_]+)\s*\(", text, re.M)))


def test_header_declares_the_shim_exports():
    assert _declared_functions() == sorted(_lib.EXPORTS)


def test_library_loads_and_exports_every_symbol():
    lib = _lib.load()
    for name in _declared_functions():
        assert hasattr(lib, name), name
    assert _lib.version() == (1, 2)
    assert _lib.launch_count() >= 0


def test_last_error_is_empty_string_initially():
    assert isinstance(_lib.last_error(), str)


def test_footprint_words_without_gpu():
    L = _lib.PkLaunch()
    L.family = _lib.FAMILY_IDS["reverse"]
    L.variant = _lib.VARIANT_STAGED
    L.s, L.B, L.N = 4, 256, 1 << 20
    assert _lib.footprint_words(L) == 1024  # the case's s*B words
    L.variant = _lib.VARIANT_DIRECT
    assert _lib.footprint_words(L) == 0


def _c_layout(struct: str, fields):
    src = ["#include <stdio.h>", "#include <stddef.h>", '#include "pk.h"', "int main(void){"]
    src.append('printf("%%zu\\n", sizeof(%s));' % struct)
    for f in fields:
        src.append('printf("%%zu\\n", offsetof(%s, %s));' % (struct, f))
    src.append("return 0;}")
    return "\n".join(src)


@pytest.mark.parametrize("struct,cls", [("pk_launch_t", _lib.PkLaunch), ("pk_machine_t", _lib.PkMachine)])
def test_ctypes_layout_matches_header(tmp_path, struct, cls):
    fields = [f for f, _ in cls._fields_]
    c = tmp_path / "layout.c"
    c.write_text(_c_layout(struct, fields))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(REPO, "include"), str(c), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    assert got[0] == ctypes.sizeof(cls)
    assert got[1:] == [getattr(cls, f).offset for f in fields]


def test_status_codes_map_to_reference_exceptions():
    # pk.h codes -> the exceptions parakern.interp raises (interp.py:75, 209-212, 43-46)
    for rc, exc in [(_lib.PK_E_PARAM, ValueError), (_lib.PK_E_BOUNDS, IndexError),
                    (_lib.PK_E_DIV0, ZeroDivisionError), (_lib.PK_E_UNSUPPORTED, NotImplementedError),
                    (_lib.PK_E_ALLOC, MemoryError), (_lib.PK_E_CUDA, _lib.PkError)]:
        with pytest.raises(exc):
            _lib.check(rc)


def _launch(family, **kw):
    L = _lib.PkLaunch()
    L.family = _lib.FAMILY_IDS[family]
    L.variant = _lib.VARIANT_STAGED
    for k, v in kw.items():
        setattr(L, k, v)
    return L


@pytest.mark.parametrize("family,kw,need", [
    # reverse N=100, s*B=64: a[0..63] read, c[36..99] written
    ("reverse", dict(N=100, s=2, B=32), [64, 100]),
    ("reverse", dict(N=100, s=2, B=32, lo=8, hi=16), [16, 92]),
    # transpose N=10, I = 9 rows (B0=3), J = 8 cols (s*B1=4): c[8*10+7], a[7][8]
    ("transpose", dict(N=10, s=2, B0=3, B1=2), [7 * 10 + 9, 8 * 10 + 8]),
    ("matvec", dict(N=10, s=1, B=4), [80, 10, 8]),
    ("matmul", dict(N=10, B0=4, ub1=3, s=1), [7 * 10 + 8, 7 * 10 + 9, 7 * 10 + 9]),
    ("addition", dict(N=8, B0=3, B1=2), [5 * 8 + 8, 5 * 8 + 8, 5 * 8 + 8]),
    ("jacobi", dict(N=10, T=2, s=2, B=2), [20]),
    ("jacobi", dict(N=10, T=0, s=2, B=2), [0]),
    ("reverse", dict(N=100, s=-1, B=32), [0, 0]),
])
def test_required_elems_without_gpu(family, kw, need):
    """pk_required_elems: 1 + the largest flat index the run touches (host-only)."""
    assert _lib.required_elems(_launch(family, **kw), len(need)) == need


def test_launch_checked_raises_index_error_before_launching():
    """pk_launch_checked refuses short buffers with PK_E_BOUNDS (the
    reference's IndexError, interp.py:209-212) before touching a device, so
    it runs here without a GPU."""
    L = _launch("reverse", N=100, s=2, B=32)
    with pytest.raises(IndexError, match=r"c\[99\]"):
        _lib.launch_checked(L, [0x1000, 0x2000], [100, 99])
    with pytest.raises(IndexError, match=r"a\[63\]"):
        _lib.launch_checked(L, [0x1000, 0x2000], [63, 100])
    with pytest.raises(ZeroDivisionError):
        _lib.launch_checked(_launch("reverse", N=100, s=0, B=32), [0x1000, 0x2000], [100, 100])
    with pytest.raises(IndexError):
        _lib.run_host(L, [0x1000, 0x2000], 0, elems=[100, 64])


def test_required_elems_match_reference_index_errors():
    """The shortest 1-D arrays the reference interpreter runs on without an
    IndexError (tests/golden/make_values.py) == pk_required_elems."""
    import json

    with open(os.path.join(REPO, "tests", "golden", "value_vectors.json")) as fh:
        bounds = json.load(fh)["bounds"]
    from paper_1801_04348_b200 import binding, programs

    for b in bounds:
        if b["family"] == "jacobi":
            continue  # the C ABI asks for the whole double buffer; the shim checks N+P+2 (GPU test)
        kind = programs.original(b["family"])
        L = binding.make_launch(kind, b["params"], ())
        names = [a.name for a in programs.FAMILIES[b["family"]].arrays]
        need = dict(zip(names, _lib.required_elems(L, len(names))))
        for name, n in b["min_len"].items():
            assert need[name] == n, (b, name)
