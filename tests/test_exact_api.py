"""The rebuilt exact-arithmetic and builder helpers (exact.py, transforms.py) keep the
reference's contracts: rounding edge cases, polynomial algebra, point parsing,
Chebyshev nodes, multiplication counts, integer forms.  Known answers here; the
same calls against the live reference when /root/reference is mounted."""
import sys
from fractions import Fraction

import numpy as np
import pytest

import _golden as G
import paper_1803_10986_b200 as W
from paper_1803_10986_b200 import exact as E
from paper_1803_10986_b200 import transforms as T


def _ref():
    if not G.reference_available():
        pytest.skip("reference not mounted")
    if G.REFERENCE_SRC not in sys.path:
        sys.path.insert(0, G.REFERENCE_SRC)
    import toomcook
    return toomcook


EDGE = [Fraction(0), Fraction(1, 3), Fraction(-2, 3), Fraction(1, 10), Fraction(2 ** 128 - 2 ** 104),
        Fraction(2 ** 128 - 2 ** 103 - 1), Fraction(1, 2 ** 149), Fraction(3, 2 ** 150), Fraction(1, 2 ** 150),
        Fraction(2 ** 24 + 1), Fraction(2 ** 24 + 3), Fraction(2 ** 53 + 1), Fraction(7, 2 ** 1076),
        Fraction(-(2 ** 1024 - 2 ** 971)), Fraction(123456789, 1000)]


def test_to_nearest_float_edges():
    assert E.to_nearest_float(Fraction(2 ** 24 + 1), "fp32") == np.float32(2 ** 24)        # tie to even
    assert E.to_nearest_float(Fraction(2 ** 24 + 3), "fp32") == np.float32(2 ** 24 + 4)
    assert E.to_nearest_float(Fraction(1, 2 ** 150), "fp32") == np.float32(0.0)              # half of min subnormal
    assert E.to_nearest_float(Fraction(3, 2 ** 150), "fp32") == np.float32(2.0 ** -148)
    with pytest.raises(OverflowError):
        E.to_nearest_float(Fraction(2 ** 128 - 2 ** 103), "fp32")
    assert E.to_nearest_float(Fraction(2 ** 128 - 2 ** 103 - 1), "fp32") == np.finfo(np.float32).max
    with pytest.raises(ValueError):
        E.to_nearest_float(Fraction(1), "fp16")
    for v in EDGE:
        for prec in ("fp32", "fp64"):
            try:
                got = E.to_nearest_float(v, prec)
            except OverflowError:
                continue
            assert Fraction(float(got)) == Fraction(float(np.asarray(float(v) if prec == "fp64" else got)))


def test_to_nearest_float_vs_reference():
    tc = _ref()
    for v in EDGE + [Fraction(k, 7 ** j) for k in range(-50, 50, 7) for j in range(1, 30, 4)]:
        for prec in ("fp32", "fp64"):
            if prec == "fp32" and Fraction(2 ** 128 - 2 ** 104) < abs(v) < Fraction(2 ** 128 - 2 ** 103):
                # below the documented threshold the reference narrows a binary64 value that
                # already rounded up to 2^128 - 2^103 and overflows on the way (exact.py:76-79);
                # the correctly rounded answer is the largest binary32 (test above)
                continue
            try:
                want = tc.exact.to_nearest_float(v, prec)
            except OverflowError:
                with pytest.raises(OverflowError):
                    E.to_nearest_float(v, prec)
                continue
            got = E.to_nearest_float(v, prec)
            assert type(got) is type(want) and got.tobytes() == want.tobytes(), (v, prec)


def test_polynomials_and_points():
    p = E.poly_product([E.Polynomial.from_root(r) for r in (1, -1, Fraction(1, 2))])
    assert p.coeffs == (Fraction(1, 2), -1, Fraction(-1, 2), 1)
    assert p.evaluate(Fraction(1, 2)) == 0 and p.evaluate(2) == 3 * 1 * Fraction(3, 2)
    assert p.deflate(1) == E.Polynomial.from_roots([-1, Fraction(1, 2)])
    assert (E.Polynomial([1, 1]) * E.Polynomial([0, 0, 2])).coeffs == (0, 0, 2, 2)
    assert E.Polynomial([0, 0]).coeffs == () and p.padded(6)[4:] == (0, 0)
    with pytest.raises(ValueError):
        p.padded(2)
    with pytest.raises(ValueError):
        E.poly_product([])
    pts = E.parse_points(" 0, -1, 1/2, −4/3 ,inf,")
    assert [str(q) for q in pts] == ["0", "-1", "1/2", "-4/3", "inf"]
    assert pts[-1] is E.INFINITY or pts[-1] == E.INFINITY
    assert sorted(pts, key=lambda q: q.sort_key())[0].value == Fraction(-4, 3)
    for bad in ("", "1/0", "x", "1.5"):
        with pytest.raises(ValueError):
            E.parse_points(bad) if bad in ("",) else E.parse_point(bad)
    with pytest.raises(ValueError):
        E.validate_point_set(E.parse_points("0,1,0"))
    with pytest.raises(ValueError):
        E.validate_point_set(E.parse_points("0,inf,oo"))
    import pickle
    assert pickle.loads(pickle.dumps(pts)) == pts


def test_builder_helpers_vs_reference():
    tc = _ref()
    for n in range(1, 12):
        a = W.chebyshev_points(n)
        b = tc.transforms.chebyshev_points(n)
        assert [q.value for q in a] == [q.value for q in b]
    for nh, no, d in ((3, 2, 1), (3, 6, 2), (5, 4, 2)):
        x, y = W.mult_count(nh, no, d), tc.transforms.mult_count(nh, no, d)
        assert (x.general_mults, x.mults_per_output) == (y.general_mults, y.mults_per_output)
    for text in ("0,1,-1,inf", "0,-1,1,1/2,-1/2,2,-2,inf", "0,1,-1,2,-2", "3,1/3,-5/7"):
        pts = W.parse_points(text)
        r = 3 if len(pts) >= 3 else 2
        ours = W.build_transforms(r, len(pts) - r + 1, pts)
        ref = tc.build_transforms(r, len(pts) - r + 1, tc.parse_points(text))
        assert ours.square_a_t() == ref.square_a_t()
        for name in ("A_T", "G", "B_T"):
            oi, od = ours.int_form(name)
            ri, rd = ref.int_form(name)
            assert od == rd and (oi == ri).all()
        assert ours.to_json_dict() == ref.to_json_dict() and repr(ours) == repr(ref)
    for nh, no in ((3, 2), (2, 2), (1, 3)):
        with pytest.raises(ValueError):
            T.build_toom_cook(nh, no, W.parse_points("0,1,-1,inf")[: nh + no - 1] + (E.INFINITY,))
