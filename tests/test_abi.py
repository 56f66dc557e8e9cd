"""CPU checks of the boundary: the C-ABI library loads without a GPU, exports
every symbol include/mf.h declares, the binding wraps each of them, and the
product package never touches the oracle."""
import ast
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mf.h")
PKG = os.path.join(ROOT, "paper_1910_13247_b200")


def declared():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:mf_status|void|const char \*)\s*(mf_\w+)\s*\(", txt, re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_1910_13247_b200 import build, mf

    build.build()
    return mf.load()


def test_header_declares_the_boundary():
    names = declared()
    for n in ["mf_create", "mf_apply", "mf_diagonal", "mf_cg_solve", "mf_destroy", "mf_apply_host",
              "mf_estimate_lambda_max", "mf_chebyshev", "mf_sizes"]:
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.check_output(["nm", "-D", "--defined-only", os.path.join(PKG, "libmf_b200.so")]).decode()
    exported = set(re.findall(r" T (mf_\w+)", out))
    missing = set(declared()) - exported
    assert not missing, missing
    for n in declared():
        assert hasattr(lib, n)


def test_binding_wraps_every_symbol():
    from paper_1910_13247_b200 import mf

    assert sorted(mf.EXPORTS) == declared()


def test_library_is_sm100a():
    so = os.path.join(PKG, "libmf_b200.so")
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so]).decode()
    assert "sm_100a" in out


def test_error_path_without_gpu(lib):
    # argument validation happens before any CUDA call
    import ctypes

    from paper_1910_13247_b200 import mf

    m = mf.Mesh()
    m.dim = 4
    c = mf.Coeff(0, 1.0)
    h = ctypes.c_void_p()
    code = lib.mf_create(ctypes.byref(m), 2, ctypes.byref(c), None, ctypes.byref(h))
    assert code == -1 and b"dim" in lib.mf_last_error()
    m.dim = 3
    for e in range(3):
        m.n_cells[e] = 2
        m.upper[e] = 1.0
    code = lib.mf_create(ctypes.byref(m), 9, ctypes.byref(c), None, ctypes.byref(h))
    assert code == -1 and b"degree" in lib.mf_last_error()


def test_product_never_imports_oracle():
    for dirpath, _, files in os.walk(PKG):
        for f in files:
            p = os.path.join(dirpath, f)
            if f.endswith(".py"):
                tree = ast.parse(open(p).read())
                for node in ast.walk(tree):
                    if isinstance(node, ast.Import):
                        assert all(not a.name.startswith("oracle") for a in node.names), p
                    if isinstance(node, ast.ImportFrom):
                        assert not (node.module or "").startswith("oracle"), p
            if f.endswith((".cu", ".cpp", ".h")):
                assert "oracle" not in open(p).read().replace("oracle/", "").lower() or f == "tables.cpp", p


def test_operator_refuses_without_cuda():
    import torch

    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    from paper_1910_13247_b200 import Operator

    with pytest.raises(RuntimeError, match="CUDA"):
        Operator((2, 2, 2), 2)
