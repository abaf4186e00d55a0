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


def _magic(d):
    """udiv_magic_host (csrc/ctf_filter.cu): s = floor(log2 d), m = ceil(2^(32+s) / d), 0 when d
    is a power of two."""
    s = d.bit_length() - 1
    m = 0 if d & (d - 1) == 0 else -(-(1 << (32 + s)) // d)
    return m, s


def _udiv(n, m, s):
    return ((n * m) >> 32 if m else n) >> s


def test_udiv_magic_is_exact():
    """The kernels' magic-number division (frames, wave-rows, runs of a row) equals n // d for
    every divisor they use and numerators below 2^31 (edges and a random sample)."""
    import random
    rnd = random.Random(5)
    ds = list(range(1, 2049)) + [3 * 1024, 4095, 4096, 4097, 259200, 64800, 16588800, (1 << 20) + 1]
    for d in ds:
        m, s = _magic(d)
        ns = {0, 1, d - 1, d, d + 1, 2 * d - 1, (1 << 31) - 1, (1 << 31) - d}
        ns |= {rnd.randrange(0, 1 << 31) for _ in range(40)}
        for n in ns:
            if 0 <= n < (1 << 31):
                assert _udiv(n, m, s) == n // d, (n, d)


def test_equal_runs_partition_a_row():
    """Lean-kernel runs (launch_fast / the kernel's run bounds): run j of a wave-row spans waves
    [j nwx / cpr, (j+1) nwx / cpr); for every cpr the launcher can pick (ceil(nwx / 16) ..
    max(nwx / 2, that)) the runs cover the row exactly once, lengths differ by at most one and
    never exceed 16 waves (nor fall below 2 when cpr <= nwx / 2)."""
    for nwx in list(range(1, 130)) + [240, 480, 481, 2048]:
        rmin = -(-nwx // 16)
        rmax = max(nwx // 2, rmin)
        for cpr in sorted({rmin, rmax, (rmin + rmax) // 2}):
            m, s = _magic(cpr)
            bounds = [_udiv(j * nwx, m, s) for j in range(cpr + 1)]
            assert bounds[0] == 0 and bounds[-1] == nwx
            lens = [b - a for a, b in zip(bounds, bounds[1:])]
            assert max(lens) - min(lens) <= 1 and max(lens) <= 16
            if cpr <= nwx // 2:
                assert min(lens) >= 2


def test_vertical_band_item_order_is_a_bijection():
    """run_coords (CTF_VBAND = 8): work item rr of a frame -> (wave-row, run column) runs down
    bands of 8 wave-rows first; every (row, column) of the frame is hit exactly once, including
    the last, shorter band."""
    B = 8
    for nwy in (1, 3, 8, 9, 17, 270, 540):
        for cpr in (1, 2, 5, 30):
            seen = set()
            for rr in range(nwy * cpr):
                bs = B * cpr
                band, q = rr // bs, rr % bs
                h = min(B, nwy - band * B)
                wxc = q // h
                wy = band * B + (q - wxc * h)
                assert 0 <= wy < nwy and 0 <= wxc < cpr
                seen.add((wy, wxc))
            assert len(seen) == nwy * cpr
