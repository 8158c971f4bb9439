"""CPU checks of the boundary: libwbfbt.so loads (no GPU needed -- cudart is
linked statically) and exports every entry point include/wbfbt.h declares;
the binding's SYMBOLS table matches the header exactly; the product package
never imports the oracle."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "wbfbt.h")


def _header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(wb_[a-z_A-Z0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def built():
    from paper_1607_03936_b200 import build
    return build.build()


def test_header_declares_the_section8b_calls():
    fns = _header_functions()
    for need in ["wb_create", "wb_destroy", "wb_sizes", "wb_set_viscosity", "wb_apply_A", "wb_apply_B",
                 "wb_apply_BT", "wb_apply_K", "wb_poisson_pcg", "wb_apply_wbfbt", "wb_debug_pcg_step",
                 "wb_get_dofmap", "wb_get_boundary_mask", "wb_get_lumped", "wb_query", "wb_sync",
                 "wb_last_error"]:
        assert need in fns


def test_library_exports_every_header_symbol(built):
    L = ctypes.CDLL(built)
    for name in _header_functions():
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", built], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (wb_\w+)", out))
    assert exported == set(_header_functions())


def test_binding_table_matches_header(built):
    from paper_1607_03936_b200 import SYMBOLS, lib, version
    assert sorted(n for n, _, _ in SYMBOLS) == _header_functions()
    lib()
    assert "sm_100a" in version()


def test_library_is_sm100a_only(built):
    out = subprocess.run(["cuobjdump", "--list-elf", built], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1607_03936_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle", txt, re.M), f
                assert "liboracle" not in txt and "oracle.c" not in txt, f


def test_create_without_gpu_fails_loudly(built):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1607_03936_b200 import lib
    h = ctypes.c_void_p()
    st = lib().wb_create(ctypes.byref(h), 4, 2, 0, None)
    assert st != 0 and not h.value


def test_every_option_and_query_key_is_documented():
    """Every key wb_set_option accepts, and every key wb_query answers, is named in the
    header's documentation (include/wbfbt.h), so the ABI description stays complete."""
    import re
    src = open(os.path.join(ROOT, "paper_1607_03936_b200", "csrc", "wbfbt.cu")).read()
    hdr = open(os.path.join(ROOT, "include", "wbfbt.h")).read()
    i, j = src.index("wb_status wb_set_option("), src.index("wb_status wb_sync(")
    opts = re.findall(r'strcmp\(key, "([^"]+)"\)', src[i:j])
    assert len(opts) >= 10
    missing = [k for k in opts if f'"{k}"' not in hdr]
    assert not missing, f"options not documented in include/wbfbt.h: {missing}"
    i, j = src.index("wb_status wb_query("), src.index("wb_status wb_set_option(")
    keys = re.findall(r'strcmp\(key, "([^"]+)"\)', src[i:j])
    prefixes = re.findall(r'strncmp\(key, "([^"]+)"', src[i:j])
    assert len(keys) >= 10
    missing = [k for k in keys if f'"{k}"' not in hdr] + [p for p in prefixes if f'"{p}' not in hdr]
    assert not missing, f"query keys not documented in include/wbfbt.h: {missing}"
