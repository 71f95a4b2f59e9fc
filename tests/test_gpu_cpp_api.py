"""The C++ drop-in headers (include/vqkv/*.hpp) compile against the library and
pass reference-style tests on the GPU (tests/cpp/test_cpp_api.cpp)."""
import os
import subprocess

import pytest


def test_cpp_headers_compile_cpu():
    """Header-only C++ mirror builds and links (no GPU needed)."""
    from paper_2603_16435_b200 import build

    assert os.path.exists(build.build_cpp_tests())


@pytest.mark.gpu
def test_cpp_api_on_gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2603_16435_b200 import build

    exe = build.build_cpp_tests()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL" not in r.stdout
