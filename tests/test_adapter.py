"""The reference-side adapter (paper_2503_17491_b200.adapter.install) re-points every
hot-path name the reference's consumers bind (SURVEY 8(b) "Callers to patch":
mapping.py:38-44, registration.py:27, pipeline.py:30, cli.py:45) and restores them.

Runs on CPU: patching does not touch the device.  Uses the live reference when it
is importable (this container), and a stand-in package of the same layout otherwise.
"""
import importlib
import os
import sys
import textwrap

import pytest

from paper_2503_17491_b200 import adapter
from paper_2503_17491_b200 import mapping as MP
from paper_2503_17491_b200 import rasterizer as RZ
from paper_2503_17491_b200 import registration as REG

REF_SRC = "/root/reference/pkg/src"


def _check(pkg):
    orig = {(m, n): getattr(importlib.import_module(f"{pkg}.{m}"), n)
            for m, names in adapter.PATCH_TABLE.items() for n in names}
    inst = adapter.install(pkg)
    try:
        assert set(inst.patched) == set(orig)
        for (m, n), o in orig.items():
            now = getattr(importlib.import_module(f"{pkg}.{m}"), n)
            assert now is not o, (m, n)
        mod = lambda m: importlib.import_module(f"{pkg}.{m}")  # noqa: E731
        for m in ("rasterizer", "mapping", "registration", "pipeline", "cli"):
            assert mod(m).rasterize_forward is RZ.rasterize_forward
        for m in ("rasterizer", "mapping"):
            assert mod(m).rasterize_backward is RZ.rasterize_backward
        assert mod("mapping").refine is MP.refine and mod("pipeline").refine is MP.refine
        assert mod("registration").build_leaf_tree is REG.build_leaf_tree
        assert mod("registration").register is mod("pipeline").register
        assert mod("mapping").make_keyframe is mod("pipeline").make_keyframe
    finally:
        inst.uninstall()
    for (m, n), o in orig.items():
        assert getattr(importlib.import_module(f"{pkg}.{m}"), n) is o


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference not present")
def test_install_patches_live_reference():
    sys.path.insert(0, REF_SRC)
    try:
        _check("splatscan")
    finally:
        sys.path.remove(REF_SRC)


def test_install_patches_standin_package(tmp_path):
    pkg = tmp_path / "fake_splatscan"
    pkg.mkdir()
    (pkg / "__init__.py").write_text("")
    bodies = {
        "rasterizer": "def rasterize_forward(*a): pass\ndef rasterize_backward(*a): pass\n",
        "mapping": "from .rasterizer import rasterize_forward, rasterize_backward\n"
                   "class Keyframe: pass\ndef make_keyframe(*a): pass\ndef refine(*a): pass\n",
        "registration": "from .rasterizer import rasterize_forward\nclass RegistrationResult: pass\n"
                        "def register(*a): pass\ndef build_leaf_tree(*a): pass\n",
        "pipeline": "from .rasterizer import rasterize_forward\nfrom .registration import register\n"
                    "from .mapping import refine, make_keyframe\n",
        "cli": "from .rasterizer import rasterize_forward\n",
        "geometry": "class RangeImage: pass\nclass NormalImage: pass\ndef estimate_camera(*a): pass\n",
    }
    for k, v in bodies.items():
        (pkg / f"{k}.py").write_text(textwrap.dedent(v))
    sys.path.insert(0, str(tmp_path))
    try:
        _check("fake_splatscan")
    finally:
        sys.path.remove(str(tmp_path))


def test_install_rejects_other_layouts(tmp_path):
    pkg = tmp_path / "not_splatscan"
    pkg.mkdir()
    (pkg / "__init__.py").write_text("")
    for k in ("rasterizer", "mapping", "registration", "pipeline", "cli", "geometry"):
        (pkg / f"{k}.py").write_text("")
    sys.path.insert(0, str(tmp_path))
    try:
        with pytest.raises(AttributeError):
            adapter.install("not_splatscan")
    finally:
        sys.path.remove(str(tmp_path))
