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
