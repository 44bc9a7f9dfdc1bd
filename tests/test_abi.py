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
FFMA2_LINE = re.compile(r"\bFFMA2\s+([^;]*);")


def _fused_ops(sass: str) -> list:
    """Instructions that would fuse a multiply into a per-thread sum.  FFMA/DFMA
    always do.  FFMA2 is allowed only as the packed exact product
    fma.rn.f32x2(a, b, -0) == fl(a*b) (contract_template.cuh, codegen.cpp k2_mul), whose
    addend is the (-0, -0) kernel parameter: a uniform register or constant-bank operand,
    or -- e.g. when another product in the kernel takes an immediate multiplier, which
    leaves no slot for a second special operand -- a register pair that the function only
    ever loads from the parameter bank (LDC.64 Rn, c[0x0][..]) and never writes otherwise.
    Accumulators are per-thread registers written by arithmetic, so a fused sum fails
    both tests."""
    bad = [m.group(0) for m in re.finditer(r"\b(FFMA|DFMA)\b(?!2)[^;]*;", sass)]
    nodest = ("STG", "STS", "ST", "STL", "RED", "ATOMS", "BAR", "BRA", "EXIT", "ISETP", "FSETP")
    for fn in re.split(r"\n\s*Function : ", sass):
        # program-order list of (position, opcode, registers written); destination = first operand
        writes, uses = [], []
        for m in re.finditer(r"(?:@!?U?P\d+\s+)?\b([A-Z][A-Z0-9_]*(?:\.[A-Za-z0-9_]+)*)\s+([^;/]*);", fn):
            op, body = m.group(1), m.group(2)
            base = op.split(".")[0]
            d = re.match(r"R(\d+)\b", body)
            if d and base not in nodest:
                r = int(d.group(1))
                wide = 4 if ".128" in op else 2 if (".64" in op or ".WIDE" in op or base in
                                                     ("FFMA2", "FADD2", "FMUL2", "DADD", "DMUL", "DFMA")) else 1
                writes.append((m.start(), op, set(range(r, r + wide))))
            if base == "FFMA2":
                uses.append((m.start(), m.group(0), [o.strip() for o in body.split(",")]))
        by_reg = {}
        for pos, text, ops in uses:
            if len(ops) == 4 and re.match(r"^(UR\d+|c\[0x[0-9a-f]+\]\[0x[0-9a-f]+\])", ops[3]):
                continue
            mr = re.match(r"^R(\d+)\b", ops[3]) if len(ops) == 4 else None
            if not mr:
                bad.append(text)
                continue
            by_reg.setdefault(int(mr.group(1)), []).append((pos, text))
        for n, lst in by_reg.items():
            pair = {n, n + 1}
            first, last = lst[0][0], lst[-1][0]
            before = [w for w in writes if w[0] < first and w[2] & pair]
            # the definition reaching the first use must be a parameter load covering the pair (or one
            # load per half), and nothing may write the pair while the products that use it run
            reach = {}
            for w in before:
                for q in w[2] & pair:
                    reach[q] = w[1]
            inside = [w for w in writes if first <= w[0] <= last and w[2] & pair and not w[1].startswith("LDC")]
            if set(reach) != pair or not all(o.startswith("LDC") for o in reach.values()) or inside:
                bad.extend(t for _, t in lst)
    return bad


def _pack_tag(pack):
    return {"tile": None, "pack": "8,8,16,8,16,4,0,8,0,1", "scalar": "8,8,16,8,16,4,0,8,0,0"}[pack]


@pytest.mark.parametrize("prec", ["fp32", "mixed", "fp64"])
@pytest.mark.parametrize("cs", ["linear", "pairwise"])
@pytest.mark.parametrize("pack", ["tile", "pack", "scalar"])
def test_sass_gate_exact_kernels_have_no_fma(built, prec, cs, pack, gemm_tuning):
    """Exactness needs every product and sum rounded separately: FMUL/FADD
    (DMUL/DADD) or the packed exact product FFMA2(a, b, uniform -0), never a
    multiply fused into a running sum."""
    if _pack_tag(pack):
        gemm_tuning(_pack_tag(pack))
    plan = _plan(3, 4, "0,1,-1,1/2,-1/2,inf", prec, cs)
    for which in (0, 1, 2):
        sass = _sass(plan.cubin(which, 128))
        bad = _fused_ops(sass)
        assert not bad, (which, bad[:3])
    contract = _sass(plan.cubin(2, 128))
    assert "UBLKCP" in contract          # cp.async.bulk global->shared (TMA bulk copy)
    assert re.search(r"\bSYNCS\.", contract)  # mbarrier pipeline
    if pack == "pack" and prec != "fp64":
        assert "FADD2" in contract and "FFMA2" in contract
    if pack == "scalar" or prec == "fp64":
        assert "FFMA2" not in contract


@pytest.mark.parametrize("cs", ["linear", "pairwise"])
def test_sass_gate_fused_exact_kernel(built, cs):
    """The fused exact K3 + K4 kernel (wino_conv2d_fused): separately rounded products and sums
    like the unfused contraction, accumulators parked in tensor memory (STTM / LDTM), operands
    through bulk copies, and no M store (its only global stores are the outputs)."""
    plan = _plan(3, 2, "0,1,-1,inf", "fp32", cs)
    sass = _sass(plan.cubin(3, 128))
    assert not _fused_ops(sass)
    assert "FFMA2" in sass and "FADD2" in sass and "UBLKCP" in sass
    assert re.search(r"\bSTTM\b", sass) and re.search(r"\bLDTM\b", sass)   # tcgen05.st / tcgen05.ld
    assert "STG.E.128" not in sass                                          # (the unfused kernel's M stores)
    big = _plan(3, 4, "0,1,-1,1/2,-1/2,inf", "fp32", cs)                    # alpha = 6: no fused kernel
    with pytest.raises(RuntimeError):
        big.cubin(3, 128)


def test_sass_gate_rejects_fused_sums():
    assert _fused_ops("FFMA R1, R2, R3, R4 ;")
    assert _fused_ops("FFMA2 R16, R25.F32, R32.F32x2.HI_LO, R8.F32x2.HI_LO ;")
    assert _fused_ops("DFMA R2, R4, R6, R8 ;")
    assert not _fused_ops("FFMA2 R16, R25.F32, R32.F32x2.HI_LO, UR8.F32x2.HI_LO ;")
    ldc = "        /*0100*/                   LDC.64 R2, c[0x0][0x390] ;\n"
    imm = "        /*01d0*/                   FFMA2 R4, R4.F32x2.HI_LO, 0.5, R2.F32x2.HI_LO ;\n"
    assert not _fused_ops(ldc + imm)                                   # immediate multiplier, -0 parameter addend
    assert _fused_ops(imm)                                             # addend of unknown origin
    assert _fused_ops(ldc + "        /*0110*/                   FADD2 R2, R6.F32x2.HI_LO, R8.F32x2.HI_LO ;\n" + imm)
    assert _fused_ops(ldc + "        /*0110*/                   LDS.128 R0, [R9] ;\n" + imm)  # R2 rewritten by a wide load
    assert not _fused_ops("FMUL R1, R2, R3 ; FADD2 R4, R6.F32x2.HI_LO, R8.F32x2.HI_LO ; HFMA2 R5, -RZ, RZ, 0, 0 ;")


def test_tensor_core_layer_module_has_the_stack_kernels(built):
    """The tc_* layer module (NVRTC, CPU-only compile) carries the fused K4 + ReLU / max-pool kernel and,
    at 16 < alpha^2 <= 96, the warp-per-channel K1 with its shared-memory park: separately rounded
    transform arithmetic (no FMA), 16-bit park stores, 16-byte global row stores, three 256-thread blocks
    per SM without spills; alpha^2 <= 16 keeps the register-packed 8-channel kernel instead."""
    plan = _plan(3, 6, "0,-1,1,1/2,-1/2,2,-2,inf", "fp32", "pairwise", contraction="tc_bf16")
    cub = plan.cubin(0, 0)
    sass = _sass(cub)
    fns = dict((f.split()[0], f) for f in re.split(r"\n\s*Function : ", sass)[1:])
    for k in ("wino_transforms_tcs", "wino_input_tcs", "wino_transforms_tcg", "wino_output_gather_act"):
        assert k in fns, sorted(fns)
    tcs = fns["wino_input_tcs"]
    assert not FMA.search(tcs)
    assert re.search(r"\bSTS\.U16\b", tcs) and re.search(r"\bSTG\.E\.128\b", tcs) and "BAR.SYNC" in tcs
    assert "STL" not in tcs and "LDL" not in tcs
    with tempfile.NamedTemporaryFile(suffix=".cubin") as f:
        f.write(cub)
        f.flush()
        res = subprocess.run(["cuobjdump", "-res-usage", f.name], capture_output=True, text=True, check=True).stdout
    m = re.search(r"Function wino_input_tcs:\s*\n\s*REG:(\d+) .*?SHARED:(\d+)", res)
    assert m and int(m.group(1)) <= 85 and int(m.group(2)) >= 64 * 512, res[:400]
    small = _plan(3, 2, "0,1,-1,inf", "fp32", "linear", contraction="tc_bf16")
    assert "wino_input_tcs" not in _sass(small.cubin(0, 0))


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


def test_layout_picks_per_shape(built):
    """The picked blocking follows the padded-work model (wino_host.cu pick())."""
    plan = _plan(3, 6, "0,-1,1,1/2,-1/2,2,-2,inf", "fp32", "linear")
    L = plan.layout(256, 64, 224, 224, 64, 1)     # VGG-16 layer 2: K = 64 -> 64-row blocks
    assert (L.bm, L.Kp) == (64, 64)
    L = plan.layout(256, 3, 224, 224, 64, 1)      # layer 1: C = 3
    assert L.Cp <= 16
    L = plan.layout(64, 256, 28, 28, 256, 1)      # cfg3: 128 x 64 tiles
    assert (L.bm, L.bn) == (128, 64)
