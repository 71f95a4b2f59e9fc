"""SASS guard for the bit-exact kernels (CPU: reads the built library, no GPU).

ptxas (CUDA 12.9) contracts `mul.rn.f32x2` followed by `add.rn.f32x2` into one FFMA2,
even with --fmad=false, although both carry an explicit rounding mode.  One fused
multiply-add in the candidate rescoring or the residual-norm sum changes the last bit
of a score or a norm relative to the reference's separate fp32 multiply and add
(codebook.cpp:166-172), so the exact kernels must contain no FFMA2 other than the
ones written as `ptx::fma2` on purpose (the slacked window bound).
"""
import os
import re
import shutil
import subprocess
import tempfile

import pytest

from paper_2603_16435_b200 import build

LIB = os.path.join(os.path.dirname(build.__file__), "lib", "libvqkv_b200.so")
TOOLS = all(shutil.which(t) or os.path.exists(f"/usr/local/cuda/bin/{t}") for t in ("cuobjdump", "nvdisasm"))


def _tool(t):
    return shutil.which(t) or f"/usr/local/cuda/bin/{t}"


def _helper_lines():
    src = open(os.path.join(os.path.dirname(build.__file__), "csrc", "tc_ptx.cuh")).read().splitlines()
    find = lambda pat: next(i + 1 for i, l in enumerate(src) if pat in l)
    return {"add2": find('"add.rn.f32x2'), "mul2": find('"mul.rn.f32x2'), "fma2": find('"fma.rn.f32x2')}


def _packed_ops(cubin):
    # -gi: line info with inline call stacks; the innermost frame comes first
    out = subprocess.run([_tool("nvdisasm"), "-gi", cubin], capture_output=True, text=True, check=True).stdout
    cur, fresh, ops = None, True, []
    for ln in out.splitlines():
        m = re.search(r'## File "([^"]+)", line (\d+)', ln)
        if m:
            if fresh:  # the first frame of a group is the innermost one
                cur = (os.path.basename(m.group(1)), int(m.group(2)))
                fresh = False
            continue
        if ln.strip().startswith("/*"):
            fresh = True
        o = re.search(r"\b(FFMA2|FMUL2|FADD2)\s+(R\d+),\s*(R\d+)[^,]*,\s*(R\d+)", ln)
        if o:
            # (op, innermost source line, whether both multiplicands are the same register pair)
            ops.append((o.group(1), cur, o.group(3) == o.group(4)))
    return ops


@pytest.mark.skipif(not (TOOLS and os.path.exists(LIB)), reason="needs the built library and cuobjdump/nvdisasm")
@pytest.mark.parametrize("unit", ["encode_tc", "encode_exact", "decode"])
def test_no_contracted_packed_fma_in_exact_kernels(unit):
    lines = _helper_lines()
    with tempfile.TemporaryDirectory() as d:
        subprocess.run([_tool("cuobjdump"), "-xelf", f"{unit}.sm_100a.cubin", LIB], cwd=d, check=True,
                       capture_output=True)
        ops = _packed_ops(os.path.join(d, f"{unit}.sm_100a.cubin"))
    ffma2 = [(src, sq) for op, src, sq in ops if op == "FFMA2"]
    # Every FFMA2 must come from ptx::fma2.  The only intended one in these units is the window
    # bound's sum of squares (encode_tc.cu, residual update: 4 x 16 unrolled), whose line records
    # nvdisasm sometimes loses to a neighbouring hoisted instruction; those are accepted only as
    # squares (both multiplicands one register pair), and the count caps them.
    bad = [src for src, sq in ffma2 if src != ("tc_ptx.cuh", lines["fma2"]) and not sq]
    assert not bad, f"{len(bad)} FFMA2 not written as ptx::fma2 (contracted mul2+add2?): {bad[:4]}"
    # encode_tc holds two kernels (CTA-pair and single-CTA), 64 window-bound squares each
    assert len(ffma2) <= (128 if unit == "encode_tc" else 0), f"{len(ffma2)} FFMA2 in {unit}"
