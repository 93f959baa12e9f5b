"""C-ABI library checks that need no GPU: the .so loads, exports every symbol
include/eig.h declares, and its host-side logic (panel count, V2 slot count,
error strings) agrees with the readings in DESIGN.md."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "eig.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(eig_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    import paper_1207_1773_b200 as pkg
    lib = pkg.lib()
    names = _declared()
    assert "eig_hotpath" in names and "eig_he2hb" in names
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(pkg.exported_symbols())


def test_host_logic_panels_and_slots():
    import oracle
    import synth
    import paper_1207_1773_b200 as pkg
    for n, nb, K in [(256, 16, 15), (2000, 64, 31), (5000, 64, 78), (10000, 64, 156), (20000, 64, 312),
                     (64, 64, 0), (65, 64, 1), (1, 64, 0)]:
        assert pkg.num_panels(n, nb) == K          # SURVEY §8 / reading R3
    for n, nb in [(37, 5), (256, 16), (1000, 64), (2, 1)]:
        assert pkg.v2_slots(n, nb) == oracle.v2_slots(n, nb) == synth.v2_layout(n, nb)[1]


def test_error_strings():
    import paper_1207_1773_b200 as pkg
    lib = pkg.lib()
    assert lib.eig_strerror(0) == b"success"
    assert b"not implemented" in lib.eig_strerror(-1005)
    assert b"illegal" in lib.eig_strerror(-3)


def test_no_cpu_fallback_without_gpu():
    import torch
    import paper_1207_1773_b200 as pkg
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(pkg.EigError):
        pkg.Solver(0)


def test_product_package_never_imports_oracle():
    pkgdir = os.path.join(ROOT, "paper_1207_1773_b200")
    for dp, _, files in os.walk(pkgdir):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "oracle.c" not in txt, f
