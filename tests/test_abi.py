"""The C-ABI library loads and exports every symbol include/wd.h declares; the
argument checks that need no device work; the product/oracle separation."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "wd.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(wd_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_all_header_symbols():
    import __graft_entry__
    __graft_entry__.build()
    lib = C.CDLL(os.path.join(ROOT, "paper_2101_08453_b200", "libwd.so"))
    syms = header_symbols()
    assert "wd_assemble" in syms and "wd_solve" in syms and len(syms) >= 19
    for s in syms:
        assert hasattr(lib, s), s
    import paper_2101_08453_b200 as wd
    assert sorted(wd.ABI_SYMBOLS) == syms


def test_default_options_and_inval_without_device():
    import paper_2101_08453_b200 as wd
    import torch
    o = wd.default_options()
    assert (o.pre_smooth, o.post_smooth, o.max_cycles, o.coarsest_max_free) == (2, 2, 100, 4096)
    assert o.coarsen_rule == wd.RULES["coupling_cur"] and o.nranks == 1
    X = torch.zeros((2, 2, 2), dtype=torch.float64)
    with pytest.raises(wd.WDError) as e:
        wd.wd_assemble(X, X, X, (1, 1, 1))          # n1, n2 < 3
    assert e.value.code == wd.WD_E_INVAL
    X = torch.zeros((3, 4, 4), dtype=torch.float64)
    with pytest.raises(wd.WDError) as e:
        wd.wd_assemble(X, X, X, (1, -1, 1))
    assert e.value.code == wd.WD_E_INVAL and "penalty" in wd.last_error()


def test_product_and_oracle_share_nothing():
    """The CUDA path never imports or links the oracle, and vice versa."""
    prod = os.path.join(ROOT, "paper_2101_08453_b200")
    for dp, _, fs in os.walk(prod):
        for fn in fs:
            if fn.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dp, fn)).read()
                assert "oracle" not in re.sub(r"(#|//).*", "", txt).replace("oracle/", ""), fn
                assert "orc_" not in txt, fn
    txt = open(os.path.join(ROOT, "oracle", "orc.c")).read()
    assert "wd.h" not in txt and "wd_internal" not in txt
    txt = open(os.path.join(ROOT, "oracle", "__init__.py")).read()
    assert "paper_2101_08453_b200" not in txt.split('"""', 2)[2]


def _build_c_demo(out):
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    lib = os.path.join(root, "paper_2101_08453_b200")
    cmd = ["gcc", "-O2", "-std=c11", "-Wall", "-Werror", os.path.join(root, "examples", "c_api_demo.c"),
           "-I" + os.path.join(root, "include"), "-L" + lib, "-lwd", "-Wl,-rpath," + lib, "-lm",
           "-o", out]
    return subprocess.run(cmd, capture_output=True, text=True)


def test_c_api_demo_compiles_against_header(tmp_path):
    """The boundary is a plain C library: a C program using only include/wd.h
    compiles and links against libwd.so (no torch, no Python)."""
    r = _build_c_demo(str(tmp_path / "c_api_demo"))
    assert r.returncode == 0, r.stderr
