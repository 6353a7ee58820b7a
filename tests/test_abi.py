"""The C-ABI library loads and exports every symbol include/bgk.h declares (CPU, no compute)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2408_02350_b200.build import build_library
    build_library()
    from paper_2408_02350_b200 import _lib
    return _lib.load()


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "bgk.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(bgk_[a-z_]+)\s*\(", txt)))


def test_exports_every_declared_symbol(lib):
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    from paper_2408_02350_b200 import _lib
    assert sorted(_lib.EXPORTED) == syms   # the binding declares exactly the header's functions


def test_version_and_workspace_size_host_only(lib):
    import bgk_inputs as bi
    from paper_2408_02350_b200.api import make_config
    assert b"sm_100a" in lib.bgk_version()
    nb = C.c_size_t(0)
    for cfg in (bi.C1, bi.C4, bi.C5):
        c = make_config(cfg)
        assert lib.bgk_workspace_size(C.byref(c), cfg.n_particles, C.byref(nb)) == 0
        f_bytes = 8 * cfg.n_particles * cfg.n_nodes * (2 if cfg.dims == 2 else 1)
        assert nb.value > 2 * f_bytes
    # C5 fits a single 180 GB B200 comfortably
    c = make_config(bi.C5)
    lib.bgk_workspace_size(C.byref(c), bi.C5.n_particles, C.byref(nb))
    assert nb.value < 40e9


def test_invalid_configs_rejected(lib):
    import bgk_inputs as bi
    from paper_2408_02350_b200.api import make_config
    nb = C.c_size_t(0)
    for bad in (dict(Nv=1), dict(Nv=64), dict(Nv=0), dict(dims=4), dict(vmax=float("nan"))):
        cfg = bi.C1.replace(**{k: v for k, v in bad.items()})
        c = make_config(cfg)
        assert lib.bgk_workspace_size(C.byref(c), 441, C.byref(nb)) == 1
    c = make_config(bi.C1, col_range=(5, 3))
    assert lib.bgk_workspace_size(C.byref(c), 441, C.byref(nb)) == 1
    c = make_config(bi.C1)
    assert lib.bgk_workspace_size(C.byref(c), 0, C.byref(nb)) == 1


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2408_02350_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "bgk_oracle" not in txt, f
