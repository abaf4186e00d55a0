"""Host-side checks of arithmetic shortcuts the CUDA kernels take (no GPU, no oracle).

Each test restates the exact integer definition and checks that the kernel's fp32 shortcut
cannot differ from it anywhere in the domain the kernel uses it on.
"""
import math
from fractions import Fraction


def test_eq2_lane_rank_margin():
    """eq2_lane_rank (csrc/ctf_filter.cu) computes floor(num / den), Eq. 2 (R-18 iv)
    in integers, as trunc(fl((num + 1/2) / den)) with __fdividef (MUFU.RCP + FMUL: relative
    error < 2^-21 on normal operands).  For every (j, np, na) with 1 <= na <= 32,
    0 <= np < na - 1, np <= j < na, the exact (num + 1/2) / den must lie at least
    32 * 2^-21 away from the integers on both sides, so any value within that relative
    error truncates to floor(num / den)."""
    rel = 2.0 ** -21
    worst = 1.0
    for na in range(1, 33):
        for np_ in range(0, na - 1):
            for j in range(np_, na):
                num = 2 * (na - 1) * (j - np_) + (na - 1 - np_)
                den = 2 * (na - 1 - np_)
                assert 0 <= num < 2 ** 11 and 0 < den <= 62
                q = Fraction(2 * num + 1, 2 * den)
                fl = math.floor(q)
                assert fl == num // den
                # distance to the enclosing integers, against the largest absolute error
                margin = min(q - fl, fl + 1 - q)
                err = float(q) * rel + 2.0 ** -24 * float(q)   # division error + rounding of num + 1/2
                assert float(margin) > err, (j, np_, na)
                worst = min(worst, float(margin) - err)
                # the served lane rank stays in [0, na - 1]
                assert 0 <= num // den <= na - 1
    assert worst > 0.0
