"""C-ABI library: it builds, loads without a GPU and exports every symbol include/mwu.h declares
(no compute calls here)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mwu.h")


def _declared():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(mwu_[a-z_0-9]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def so():
    from paper_2307_03307_b200 import build
    return build.build()


def test_header_declares_boundary():
    names = _declared()
    for required in ["mwu_create_csr", "mwu_create_graph", "mwu_solve", "mwu_get_x", "mwu_get_stats"]:
        assert required in names


def test_library_exports_every_declared_symbol(so):
    L = ctypes.CDLL(so)
    for name in _declared():
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (mwu_[a-z_0-9]+)$", out, flags=re.M))
    assert set(_declared()) <= exported


def test_binding_names_match_header(so):
    from paper_2307_03307_b200 import mwu
    assert sorted(mwu.EXPORTS) == _declared()
    mwu.lib()  # loads without a GPU


def test_default_options_roundtrip(so):
    from paper_2307_03307_b200 import mwu
    o = mwu.default_options()
    assert o.eta_factor == 10.0 and o.max_iter == 5000 and o.tol_prose == 1 and o.max_evals == 200
    assert o.use_graph == 1 and o.world == 1


def test_sm100a_sass(so):
    """The library carries sm_100a SASS (no PTX-JIT fallback for other archs)."""
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_oracle_in_product_path():
    """The product package never imports the oracle (the oracle is test infrastructure)."""
    pkg = os.path.join(ROOT, "paper_2307_03307_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
