"""CPU-side checks of the native boundary: libwino.so loads, exports every
symbol include/wino.h declares, and its generated sm_100a code honours the
exactness contract (no fused multiply-add in exact kernels) -- all without a GPU
(NVRTC compiles here; nothing is launched)."""

import os
import re
import shutil
import subprocess
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "wino.h")
LIB = os.path.join(ROOT, "paper_1803_10986_b200", "libwino.so")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(wino_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def built():
    if not os.path.exists(LIB):
        subprocess.run(["make", "-C", os.path.join(ROOT, "paper_1803_10986_b200", "csrc")], check=True)
    return LIB


def test_library_exports_every_declared_symbol(built):
    names = _declared()
    assert len(names) >= 25
    out = subprocess.run(["nm", "-D", "--defined-only", built], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (wino_[a-z0-9_]+)\b", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing


def test_ctypes_binding_covers_header(built):
    from paper_1803_10986_b200 import _native
    lib = _native.lib()
    bound = {name for name, _, _ in _native.SIGNATURES}
    assert set(_declared()) == bound
    assert lib.wino_version().decode().startswith("libwino")


def _plan(r, m, pts, prec, cs, order="huffman", contraction="exact"):
    import paper_1803_10986_b200 as W
    ts = W.build_transforms(r, m, W.parse_points(pts))
    return W.engine.get_plan(ts, W.ConvConfig(prec, order, cs), contraction)


def _sass(cubin: bytes) -> str:
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    with tempfile.NamedTemporaryFile(suffix=".cubin", delete=False) as fh:
        fh.write(cubin)
        path = fh.name
    try:
        return subprocess.run([cuobjdump, "-sass", path], capture_output=True, text=True, check=True).stdout
    finally:
        os.unlink(path)


FMA = re.compile(r"\b(FFMA2?|DFMA)\b")  # (HFMA2 RZ,RZ is the zeroing idiom)


@pytest.mark.parametrize("prec", ["fp32", "mixed", "fp64"])
@pytest.mark.parametrize("cs", ["linear", "pairwise"])
def test_sass_gate_exact_kernels_have_no_fma(built, prec, cs):
    """Exactness needs every product and sum rounded separately: FMUL/FADD
    (DMUL/DADD), never FFMA/FFMA2/DFMA."""
    plan = _plan(3, 4, "0,1,-1,1/2,-1/2,inf", prec, cs)
    for which in (0, 1, 2):
        sass = _sass(plan.cubin(which, 128))
        assert not FMA.search(sass), (which, FMA.search(sass).group(0))
    contract = _sass(plan.cubin(2, 128))
    assert "UBLKCP" in contract          # cp.async.bulk global->shared (TMA bulk copy)
    assert re.search(r"\bSYNCS\.", contract)  # mbarrier pipeline


def test_ffma_mode_uses_fma(built):
    plan = _plan(3, 2, "0,1,-1,inf", "fp32", "linear", contraction="ffma")
    assert FMA.search(_sass(plan.cubin(2, 128)))


def test_generated_source_is_straight_line_and_deterministic(built):
    p1 = _plan(3, 6, "0,-1,1,1/2,-1/2,2,-2,inf", "fp32", "linear")
    p2 = _plan(3, 6, "0,-1,1,1/2,-1/2,2,-2,inf", "fp32", "linear")
    s1, s2 = p1.source(0), p2.source(0)
    assert s1 == s2
    assert "__fmul_rn" in s1 and "__fadd_rn" in s1
    body = s1.split("void input_body")[1].split("} else {", 1)[1].split("__syncthreads", 1)[0]
    assert "__ldg" in body and "for (" not in body  # the transform is fully unrolled straight-line code


def test_invalid_programs_rejected(built):
    import ctypes
    from paper_1803_10986_b200 import _native
    # a program whose ADD underflows the stack
    bad = ([0, 1], [(1, -1, 0.0)], 3)
    good_g = ([0, 1, 2, 3, 4], [(0, 0, 1.0), (0, 1, 1.0), (0, 2, 1.0), (0, 2, 1.0)], 3)
    with pytest.raises(ValueError):
        _native.Plan(3, 2, "fp32", "linear", "exact", bad, bad, bad)
    with pytest.raises(ValueError):
        _native.Plan(3, 2, "fp32", "linear", "exact", good_g, good_g, good_g)  # wrong shapes
    assert ctypes  # silence linters


def test_layout_padding_rules(built):
    plan = _plan(3, 2, "0,1,-1,inf", "fp32", "linear")
    L = plan.layout(32, 128, 28, 28, 128, 1)
    assert (L.P, L.th, L.tw, L.Ho, L.Wo, L.T) == (16, 14, 14, 28, 28, 6272)
    assert L.Cp % 16 == 0 and L.Kp % 128 == 0 and L.Tp % 128 == 0
    assert L.u_bytes == 16 * L.Cp * L.Kp * 4 and L.v_bytes == 16 * L.Cp * L.Tp * 4
    with pytest.raises(ValueError):
        plan.layout(1, 1, 2, 2, 1, 0)  # smaller than the kernel
