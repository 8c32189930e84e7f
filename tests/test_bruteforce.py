"""Oracle vs brute-force optimal packings of tiny rectangle sets (north star:
"checked ... against brute-force optimal packings of tiny rectangle sets").

For axis-aligned rectangles every proxy is exact, so the dilated footprint of
a w x h (texel) rectangle at scale m/M is (ceil(w m/M) + 2g) x (ceil(h m/M) + 2g)
(D11, D13).  The exhaustive search places those boxes (either orientation,
P:1036 "multiple-of-90 rotations") at normal-pattern positions inside the
dilated atlas (W + 2g) x (H + 2g).  Feasibility is monotone in m, so m_opt is
the largest feasible m.  TABI is a heuristic: m_TABI <= m_opt always, with
equality on constructed cases where greedy rows are optimal.
"""
import math
from fractions import Fraction

import pytest

import chartgen

M = 64


def _boxes(rects, m, g):
    return [(math.ceil(Fraction(w * m, M)) + 2 * g, math.ceil(Fraction(h * m, M)) + 2 * g)
            for w, h in rects]


def feasible(boxes, Wp, Hp):
    boxes = sorted(boxes, key=lambda b: -b[0] * b[1])
    placed = []

    def fits(x, y, w, h):
        if x + w > Wp or y + h > Hp:
            return False
        for (px, py, pw, ph) in placed:
            if x < px + pw and px < x + w and y < py + ph and py < y + h:
                return False
        return True

    def rec(i):
        if i == len(boxes):
            return True
        xs = sorted({0} | {p[0] + p[2] for p in placed})
        ys = sorted({0} | {p[1] + p[3] for p in placed})
        seen = set()
        for (w, h) in (boxes[i], boxes[i][::-1]):
            if (w, h) in seen:
                continue
            seen.add((w, h))
            for x in xs:
                for y in ys:
                    if fits(x, y, w, h):
                        placed.append((x, y, w, h))
                        if rec(i + 1):
                            return True
                        placed.pop()
        return False

    return rec(0)


def m_opt(rects, W, H, g):
    for m in range(M, 0, -1):
        if feasible(_boxes(rects, m, g), W + 2 * g, H + 2 * g):
            return m
    return 0


def _pack(orc, rects, W, H, g):
    polys = [[(0, 0), (w, 0), (w, h), (0, h)] for (w, h) in rects]
    polys = [[(x + 10 * i, y + 3 * i) for (x, y) in p] for i, p in enumerate(polys)]
    cs = chartgen.from_polygons(polys, W, H, gutter=g)
    st, pl, info, _ = orc.pack(cs)
    if st == orc.OK:
        assert orc.validate(cs, pl) == {"overlap": 0, "gutter": 0, "oob": 0}
    return info.scale_index if st == orc.OK else 0


# cases where one greedy row / row-stack is optimal (hand-argued in comments)
EXACT = [
    # 4 squares of 40 in 64^2, g=1: 2x2 tiling needs ceil(40s) <= 31 -> m <= 49;
    # at m = 50 each box is 34 wide and 4*34^2 > 66^2.
    ([(40, 40)] * 4, 64, 64, 1, 49),
    # 2 squares of 48: side by side needs 2*(ceil(48s)+2) <= 66 -> m <= 41; at 42
    # each box is 34 > 33 in both axes so no two fit.
    ([(48, 48)] * 2, 64, 64, 1, 41),
    # 3 squares of 40: at m = 50 (34-boxes) no two fit; m = 49 -> 2 + 1 rows.
    ([(40, 40)] * 3, 64, 64, 1, 49),
    # one row of equal-height rectangles that exactly fills the width at m = 64
    ([(20, 30), (20, 30), (22, 30)], 62, 40, 0, 64),
]


@pytest.mark.parametrize("case", EXACT, ids=lambda c: f"{len(c[0])}rects")
def test_exact_cases(orc, case):
    rects, W, H, g, expect = case
    assert m_opt(rects, W, H, g) == expect
    assert _pack(orc, rects, W, H, g) == expect


@pytest.mark.parametrize("seed", range(24))
def test_random_tiny_upper_bound(orc, seed):
    rng = chartgen.SplitMix64(1234 + seed)
    n = rng.randint(2, 5)
    rects = [(rng.randint(6, 44), rng.randint(6, 44)) for _ in range(n)]
    W, H, g = rng.randint(40, 72), rng.randint(40, 72), rng.randint(0, 1)
    mt = _pack(orc, rects, W, H, g)
    mo = m_opt(rects, W, H, g)
    assert mt <= mo
    assert mo >= 1
