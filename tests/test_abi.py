"""CPU-side checks of the boundary: libtqp.so builds, loads, and exports every
function include/tqp.h declares; the binding's signature table covers them all.
No compute calls (no GPU here)."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "tqp.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b(tqp_[a-z0-9_]+)\s*\(", src)
    return sorted(set(names))


def test_header_declares_the_north_star_operators():
    names = declared_functions()
    for op in ["tqp_sort", "tqp_pkfk_join", "tqp_smj_join", "tqp_groupby_agg", "tqp_filter_compact"]:
        assert op in names


def test_library_builds_and_exports_every_declared_symbol():
    from paper_2203_01877_b200 import build as B
    lib_path = B.build()
    lib = ctypes.CDLL(lib_path)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    assert lib.tqp_abi_version() == 1


def test_binding_covers_every_symbol():
    import paper_2203_01877_b200 as T
    assert sorted(T.EXPORTED) == declared_functions()


def test_struct_layouts_match_header():
    import paper_2203_01877_b200 as T
    assert ctypes.sizeof(T.Col) == 16
    assert ctypes.sizeof(T.Pred) == 16
    assert ctypes.sizeof(T.Agg) == 56                      # static_assert'ed in csrc/api.cu


def test_binding_refuses_cpu_only():
    import torch
    import paper_2203_01877_b200 as T
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        T.Context()


def test_oracle_and_product_share_nothing():
    """The oracle imports nothing from the product package and vice versa."""
    osrc = open(os.path.join(ROOT, "oracle", "oracle.c")).read() + open(os.path.join(ROOT, "oracle", "__init__.py")).read()
    assert not re.search(r"^\s*(import|from)\s+paper_2203_01877_b200", osrc, re.M)
    assert not re.search(r"#include\s+[<\"].*tqp", osrc)
    for dp, _, fs in os.walk(os.path.join(ROOT, "paper_2203_01877_b200")):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                s = open(os.path.join(dp, f)).read()
                assert "import oracle" not in s and "from oracle" not in s and "oracle.c" not in s, f
