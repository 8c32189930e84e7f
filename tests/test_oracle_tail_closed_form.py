"""Closed-form pin of the oracle's hybrid prefix tail (D23-D26; P:316-323
"Performance Optimization", P:141 FastAtlas' intermediate downscaling; DESIGN.md
R3).

For n equal axis-aligned a x a squares and a threshold t_opt above their height,
every chart goes to the prefix tail at the first row (D23: "when no more knees
are detected and the height of the tallest chart in the row decreases below a
threshold t_opt").  Squares never interlock, so the compaction advance
of every pair is the dilated width Wd = ceil(a m / M) + 2g, and everything the
tail computes has a closed form derived here from the paper's steps -- not from
the oracle's code:
  * prefix rows: start(c) = c Wd, row q = floor(start / W') ("the prefix sum
    of the horizontal offsets"; D24);
  * the widest row extent E = (charts in the fullest row) x Wd;
  * the intermediate scale p / 2^20 = floor(m 2^20 W' / (M E)), never above
    m 2^20 / M ("intermediate scaling down", R3);
  * re-layout rounds: at p the squares' width is ceil(a p / 2^20) + 2g, the row
    partition is kept, and while the widest row still exceeds W' the scale
    shrinks by W' / E' (at most 8 rounds);
  * success iff the rows stack within H' (flat rows of equal squares);
  * the winner maximises the area-weighted mean final scale (D25): with
    every chart in the tail that is the largest p, ties to the larger m;
  * the stretch is the uniform scale's 2^20 / p (D26).
A mistake in the oracle's scan, row assignment, E, the sigma formula, its cap,
the rounds or the choice shows up as a mismatch in some candidate's (success,
p, prefix rows) or in the winner.  The cases include the cap binding (a single
short row, sigma = 1) and rows whose counts alternate (32 / 33 charts).
"""
import math
from fractions import Fraction

import pytest

import chartgen

P20 = 1 << 20


def closed_form(a, n, W, H, g, M, rounds=8):
    Wp, Hp = W + 2 * g, H + 2 * g
    out = {}
    for m in range(1, M + 1):
        Wd = math.ceil(Fraction(a * m, M)) + 2 * g
        if Wd > Wp:
            out[m] = (False, 0, 0)
            continue
        counts = {}
        for c in range(n):
            q = (c * Wd) // Wp
            counts[q] = counts.get(q, 0) + 1
        fullest = max(counts.values())
        p = min((m * P20 * Wp) // (M * fullest * Wd), (m * P20) // M)
        ok = p >= 1
        it = 0
        while ok:
            Ep = fullest * (math.ceil(Fraction(a * p, P20)) + 2 * g)
            if Ep <= Wp:
                break
            if it >= rounds:
                ok = False
                break
            p = (p * Wp) // Ep
            it += 1
            ok = p >= 1
        rows = len(counts)
        if ok:
            ok = rows * (math.ceil(Fraction(a * p, P20)) + 2 * g) <= Hp
        out[m] = (ok, p, rows)
    return out


CASES = [(30, 400, 1024, 1, 64),   # rows of 32 / 33 squares: E > W', two rounds
         (25, 300, 1024, 1, 64),   # W' = 38 Wd exactly: E = W', sigma = 1
         (30, 10, 1024, 1, 64),    # one short row: the cap sigma <= 1 binds (R3)
         (17, 700, 512, 2, 32),    # g = 2, M = 32
         (40, 150, 1024, 0, 64),   # no gutter
         (9, 900, 256, 1, 16)]     # tight: the winner far below M


@pytest.mark.parametrize("a,n,W,g,M", CASES)
def test_prefix_tail_of_equal_squares(orc, a, n, W, g, M):
    polys = [[(0, 0), (a, 0), (a, a), (0, a)] for _ in range(n)]
    cs = chartgen.from_polygons(polys, W, W)
    want = closed_form(a, n, W, W, g, M)
    st, pl, info, cands = orc.pack(cs, with_cands=True, t_opt_bp=1000, gutter=g, scale_count=M)
    for m in range(1, M + 1):
        c = cands[m - 1]
        ok, p, rows = want[m]
        assert bool(c.success) == ok, m
        if ok:
            assert (c.switched_at, c.p, c.prefix_rows) == (0, p, rows), m
    best_p, best_m = max(((want[m][1], m) for m in want if want[m][0]), default=(0, 0))
    assert st == orc.OK and info.scale_index == best_m
    assert info.rows == 0 and info.prefix_rows == want[best_m][2]
    assert set(pl["mode"].tolist()) == {1}
    assert set(pl["scale_num"].tolist()) == {best_p} and set(pl["scale_den"].tolist()) == {P20}
    assert info.l2_stretch == pytest.approx(P20 / best_p, rel=1e-12)
    assert orc.validate(cs, pl, gutter=g) == {"overlap": 0, "gutter": 0, "oob": 0}
