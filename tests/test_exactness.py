"""Proof by exhaustion of the division-free float64 sequences the kernels use
(no GPU needed: exact rational arithmetic emulates IEEE round-to-nearest and fma).

dequantize (transform.py:122) computes RN(q / L). The kernels compute
    q0 = RN(q * r), e = fma(-q0, L, q), res = fma(e, r, q0),  r = RN(1 / L)
which must equal RN(q / L) for every representable sample q in [0, L].
"""

from fractions import Fraction as F

import pytest


def _rn(x: F) -> float:
    return float(x)  # Fraction -> float rounds to nearest-even


@pytest.mark.parametrize("B", [8, 10, 12, 16])
def test_reciprocal_division_is_exact(B):
    L = (1 << B) - 1
    r = _rn(F(1, L))
    FL, Fr = F(L), F(r)
    for q in range(L + 1):
        q0 = _rn(F(q) * Fr)
        e = _rn(F(q) - F(q0) * FL)
        got = _rn(F(e) * Fr + F(q0))
        assert got == _rn(F(q, L)), (B, q)


def test_quantize_fast_path_bound():
    """The fast path x~ = RN(RN(d*r)*L) stays within 6 ulp(L) of the reference
    x = RN(RN(d/s)*L); the kernel falls back to the exact order when x~ + 0.5 is
    within 2^-28 of an integer, far above 6 ulp(65535) = 4.4e-11."""
    ulp = 2.0 ** -52 * 65536
    assert 6 * ulp < 2.0 ** -28
