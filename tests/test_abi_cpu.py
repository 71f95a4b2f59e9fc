"""CPU-only checks of the C-ABI boundary: the library loads and exports every
symbol include/vqkv_c.h declares (no compute calls without a GPU)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "vqkv_c.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(vqkv_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_hot_path():
    syms = declared_symbols()
    for s in ("vqkv_stack_create", "vqkv_quantize_batch", "vqkv_reconstruct_block", "vqkv_attend_decode",
              "vqkv_lse_combine", "vqkv_last_error"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_2603_16435_b200 import _lib

    if not os.path.exists(_lib.LIB_PATH):
        from paper_2603_16435_b200 import build

        build.build()
    L = ctypes.CDLL(_lib.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(L, s)]
    assert not missing, missing
    # and the Python binding covers all of them
    assert set(declared_symbols()) <= set(_lib.EXPORTED)


def test_status_codes_without_gpu():
    """Validation runs before any device work, so it is testable on CPU."""
    from paper_2603_16435_b200 import _lib, errors

    L = _lib.load()
    h = ctypes.c_void_p()
    sizes = (ctypes.c_uint32 * 1)(4)
    ent = (ctypes.c_float * 8)(*([0.0] * 8))
    # zero stages -> InvalidInput (codebook.cpp:63-65)
    assert L.vqkv_stack_create(0, 0, 0, sizes, 2, ent, None, ctypes.byref(h)) == 1
    # bad kind
    assert L.vqkv_stack_create(0, 7, 1, sizes, 2, ent, None, ctypes.byref(h)) == 1
    assert b"kind" in L.vqkv_last_error()
    # non-finite entries -> InvalidInput (codebook.cpp:48-50)
    ent[3] = float("nan")
    assert L.vqkv_stack_create(0, 0, 1, sizes, 2, ent, None, ctypes.byref(h)) == 1
    with pytest.raises(errors.InvalidInput):
        _lib.call("vqkv_set_encode_path", 9)
    # lse_combine argument validation
    assert L.vqkv_lse_combine(None, None, 0, 1, 1, None, None, None) == 1


def test_cpp_reference_signatures_compile():
    """Every reference entry point binds to a pointer of the reference's signature
    (tests/cpp/test_signatures.cpp; compile-only, no GPU)."""
    import subprocess

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run(["g++", "-std=c++17", "-Wall", "-Werror", "-fsyntax-only", "-I" + os.path.join(root, "include"),
                        os.path.join(root, "tests", "cpp", "test_signatures.cpp")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
