"""The C-ABI library builds for sm_100a, loads without a GPU and exports every
symbol include/splat_b200.h declares.  CPU only (no compute calls)."""
import os
import re

from paper_2503_17491_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    txt = open(os.path.join(ROOT, "include", "splat_b200.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(ss_[a-z_0-9]+)\s*\(", txt)))


def test_library_loads_and_exports_header_symbols():
    if not os.path.exists(_lib.LIB_PATH):
        _lib.build_library()
    L = _lib.lib()
    syms = declared_symbols()
    assert len(syms) >= 10
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_lib.EXPORTED)
    assert b"sm_100a" in L.ss_version()


def test_sass_is_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
