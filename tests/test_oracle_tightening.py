"""Two-sided pins for the oracle's tightening steps (round-2 VERDICT item 1).

The earlier pins of these steps were one-sided (every covered texel lies inside
the footprint), which a looser-but-conservative bound also passes.  Here:

* hand-derived goldens (tests/golden/goldens.json, each with its citation and
  derivation): the OBB bound on a 45-degree diamond at two scales, the
  orientation's bottom-left / bottom-right branch and its odd-k middle split
  (P:459), and two hand-traced atlases that fold rows at a knee (P:304,
  Alg. 4);
* exact recomputations by a different method: the local-AABB slices (D4 + D5)
  and the OBB bound (D11) equal the extents of the polygon / of the OBB box
  clipped to each strip, computed by Sutherland-Hodgman clipping in exact
  rationals -- not by the oracle's crossing loop or its convex-minimum corner
  formula.  Both directions are checked, so a looser bound fails as well as an
  unsafe one.

Reading note (R7): D5's merge, as SURVEY §8(c) states it, is the
identity on D4's exact strip extents -- the y-band that holds a strip's topmost
point always meets the strip, so min over the meeting bands of floor(i h / k)
never exceeds the strip's own top.  The clipping test pins exactly that.
"""
import json
import math
import os
from fractions import Fraction as Fr

import numpy as np
import pytest

import chartgen

G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "goldens.json")))
U = 256
QC = [1073741824, 1053110176, 992008094, 892783698, 759250125, 596538995, 410903207, 209476638]
QS = [0, 209476638, 410903207, 596538995, 759250125, 892783698, 992008094, 1053110176]


def _proxy(orc, poly, k, flags=0):
    cs = chartgen.from_polygons([poly], 64, 64)
    st, px, bad = orc.build_proxies(cs.xy, cs.start, k, flags=flags)
    assert st == orc.OK
    return px[0]


# ---------------------------------------------------------------- goldens --

@pytest.mark.parametrize("m", [64, 32])
def test_B1_obb_bound_diamond(orc, m):
    e = G["B1_obb_diamond"]
    p = _proxy(orc, e["poly"], e["k"])
    assert p.obb_j == e["obb_j"]
    assert (p.rot90, p.fx, p.fy) == (0, 0, 0)
    pr = orc.Profile(p, m, 64, e["gutter"])
    exp = e[f"m{m}"]
    assert pr.Dtop.tolist() == exp["Dtop"]
    assert pr.Dbot.tolist() == exp["Dbot"]
    assert pr.Dleft.tolist() == exp["Dleft"]
    assert pr.Dright.tolist() == exp["Dright"]


def test_B1_without_obb_is_the_box(orc):
    """Control: the same diamond with the OBB switched off (TABI_F_NO_OBB keeps
    D6's j = 0 box) gets the plain AABB footprint -- so the golden above is
    decided by the OBB bound, not by the local slices."""
    e = G["B1_obb_diamond"]
    p = _proxy(orc, e["poly"], e["k"], flags=orc.F_NO_OBB)
    pr = orc.Profile(p, 64, 64, 0)
    assert pr.Dtop.tolist() == [0] * 9 and pr.Dbot.tolist() == [9] * 9


@pytest.mark.parametrize("name", ["O1_orient_notch_bl", "O2_orient_notch_br",
                                  "O3_orient_notch_tl", "O4_orient_middle_split"])
def test_orientation_bottom_left_right(orc, name):
    e = G[name]
    p = _proxy(orc, e["poly"], e["k"])
    assert p.rot90 == 0
    assert (p.fx, p.fy) == (e["fx"], e["fy"])


def _rect(w, h):
    return [[0, 0], [w, 0], [w, h], [0, h]]


@pytest.mark.parametrize("name", ["K1_knee_concavity", "K2_knee_margin"])
def test_knee_fold_trace(orc, name):
    e = G[name]
    W, H = e["atlas"]
    cs = chartgen.from_polygons([_rect(w, h) for w, h in e["rects"]], W, H, gutter=e["gutter"],
                                local_aabb_count=e["k"])
    st, pl, info, _ = orc.pack(cs)
    assert st == orc.OK
    assert info.scale_index == e["m"]
    assert (info.rows, info.knees_found, info.knee_rows) == (e["rows"], e["knees_found"],
                                                            e["knee_rows"])
    got = [[int(p["tx"]), int(p["ty"]), int(p["mirror_x"])] for p in pl]
    assert got == e["place"]
    assert orc.validate(cs, pl) == {"overlap": 0, "gutter": 0, "oob": 0}


# ------------------------------------------------- exact clipping (Fraction) --

def _clip(poly, a, b, axis):
    """Sutherland-Hodgman: the polygon restricted to a <= coord[axis] <= b (closed)."""
    def clip_half(pts, keep, inter):
        out = []
        n = len(pts)
        for i in range(n):
            P, Q = pts[i], pts[(i + 1) % n]
            ip, iq = keep(P), keep(Q)
            if ip:
                out.append(P)
                if not iq:
                    out.append(inter(P, Q))
            elif iq:
                out.append(inter(P, Q))
        return out

    def at(c):
        def f(P, Q):
            t = (c - P[axis]) / (Q[axis] - P[axis])
            return (P[0] + t * (Q[0] - P[0]), P[1] + t * (Q[1] - P[1]))
        return f

    pts = clip_half(poly, lambda P: P[axis] >= a, at(a))
    if not pts:
        return []
    return clip_half(pts, lambda P: P[axis] <= b, at(b))


def _floor(q: Fr) -> int:
    return q.numerator // q.denominator


def _ceil(q: Fr) -> int:
    return -((-q.numerator) // q.denominator)


def _final_pose(cs, c, p):
    """Snapped outline of chart c in its final pose (tabi.h placement steps
    1-3: translate the AABB to the origin, rot90, flips) in units."""
    a, b = int(cs.start[c]), int(cs.start[c + 1])
    q = [(int(np.rint(np.float64(cs.xy[2 * v]) * 256.0)), int(np.rint(np.float64(cs.xy[2 * v + 1]) * 256.0)))
         for v in range(a, b)]
    xs = [x for x, _ in q]
    ys = [y for _, y in q]
    q = [(x - min(xs), y - min(ys)) for x, y in q]
    w0, h0 = max(xs) - min(xs), max(ys) - min(ys)
    if p.rot90:
        q = [(h0 - y, x) for x, y in q]
    w, h = p.w, p.h
    if p.fx:
        q = [(w - x, y) for x, y in q]
    if p.fy:
        q = [(x, h - y) for x, y in q]
    return [(Fr(x), Fr(y)) for x, y in q]


def _charts(n=24):
    sets = [chartgen.generate("uv", n, 256, 256, 7, rho=0.8, side_limit=128),
            chartgen.generate("tss", n, 256, 256, 8, rho=0.8, side_limit=128),
            chartgen.generate("mixed", n, 256, 256, 9, rho=None)]
    return sets


@pytest.mark.parametrize("k", [1, 2, 3, 7, 10])
def test_slices_equal_exact_strip_extents(orc, k):
    """D4 + D5: every merged x-slice is exactly [floor(min y),
    ceil(max y)] of the final-pose polygon clipped to the closed strip
    j w / k <= x <= (j + 1) w / k, and symmetrically for y-slices.  A looser
    slice fails, and so does a merge that tightens past the polygon."""
    for cs in _charts():
        st, px, bad = orc.build_proxies(cs.xy, cs.start, k)
        assert st == orc.OK
        for c, p in enumerate(px):
            poly = _final_pose(cs, c, p)
            for j in range(k):
                part = _clip(poly, Fr(j * p.w, k), Fr((j + 1) * p.w, k), 0)
                ys = [pt[1] for pt in part]
                assert p.top[j] == _floor(min(ys)), (cs.name, c, j)
                assert p.bot[j] == _ceil(max(ys)), (cs.name, c, j)
                part = _clip(poly, Fr(j * p.h, k), Fr((j + 1) * p.h, k), 1)
                xs = [pt[0] for pt in part]
                assert p.left[j] == _floor(min(xs)), (cs.name, c, j)
                assert p.right[j] == _ceil(max(xs)), (cs.name, c, j)


def _obb_box(p):
    """The OBB region {umin <= x C + y S <= umax, vmin <= -x S + y C <= vmax}
    as an exact quadrilateral in (x, y) (inverse of the Q30 rotation)."""
    C, S = QC[p.obb_j], QS[p.obb_j]
    N = C * C + S * S
    corners = [(p.umin, p.vmin), (p.umax, p.vmin), (p.umax, p.vmax), (p.umin, p.vmax)]
    return [(Fr(u * C - v * S, N), Fr(u * S + v * C, N)) for u, v in corners]


def _rotated_rects():
    polys = []
    for i, (w, h, th) in enumerate([(40, 9, 0.39), (30, 30, 0.785), (50, 6, 0.2), (22, 61, 1.1),
                                    (35, 12, 0.6), (17, 45, 1.35), (60, 20, 0.98)]):
        c, s = math.cos(th), math.sin(th)
        pts = [(x * c - y * s, x * s + y * c) for x, y in [(0, 0), (w, 0), (w, h), (0, h)]]
        mx, my = min(x for x, _ in pts), min(y for _, y in pts)
        polys.append([[round((x - mx) * 256) / 256, round((y - my) * 256) / 256] for x, y in pts])
    return polys


@pytest.mark.parametrize("m", [64, 47, 13])
def test_obb_bound_equals_exact_box_extent(orc, m):
    """D11's OBB bound at k = 1, where the local bound is the plain
    AABB: TopEdge(i) = max(0, floor(min y)) and BottomEdge(i) = min(h_s,
    ceil(max y)) of the OBB box clipped to column i's unscaled strip (itself
    clipped to the chart extent); likewise for rows.  Covers OBB angles other
    than 0 and 4 (the rotated rectangles pick j in 1..7)."""
    M = 64
    seen = set()
    for poly in _rotated_rects():
        p = _proxy(orc, poly, 1)
        if p.obb_j == 0:
            continue
        seen.add(p.obb_j)
        box = _obb_box(p)
        SC = M * U
        pr = orc.Profile(p, m, M, 0)
        ws, hs = pr.ws, pr.hs
        for i in range(ws):
            x0, x1 = Fr(i * SC, m), min(Fr((i + 1) * SC, m), Fr(p.w))
            part = _clip(box, x0, x1, 0)
            ys = [pt[1] for pt in part]
            top = max(0, _floor(min(ys) * m / SC))
            bot = min(hs, _ceil(max(ys) * m / SC))
            assert (int(pr.Dtop[i]), int(pr.Dbot[i])) == (top, bot), (poly, m, i)
        for r in range(hs):
            y0, y1 = Fr(r * SC, m), min(Fr((r + 1) * SC, m), Fr(p.h))
            part = _clip(box, y0, y1, 1)
            xs = [pt[0] for pt in part]
            left = max(0, _floor(min(xs) * m / SC))
            right = min(ws, _ceil(max(xs) * m / SC))
            assert (int(pr.Dleft[r]), int(pr.Dright[r])) == (left, right), (poly, m, r)
    assert len(seen) >= 3, seen


@pytest.mark.parametrize("name", ["A13b_knee_update_equal_height",
                                  "A13c_knee_update_equal_height_rtl"])
def test_knee_update_equal_height(orc, name):
    """Alg. 2's comparison is >=: a texel level with the
    frontline at the knee edge moves the edge."""
    e = G[name]
    ok, left, right = orc.update_knee(e["F"], e["ltr"], e["left"], e["right"])
    assert ok == e["ok"]
    if e["ltr"]:
        assert (left, right) == (e["left"], e["new_right"])
    else:
        assert (left, right) == (e["new_left"], e["right"])


def test_knee_tie_earliest(orc):
    e = G["A17b_knee_tie_earliest"]
    assert orc.find_knee([h * U for h in e["heights"]], e["atlas_h"]) == e["knee"]


def test_sort_ties(orc):
    e = G["A25_sort_ties"]
    cs = chartgen.from_polygons([_rect(w, h) for w, h in e["rects"]], 64, 64)
    st, px, bad = orc.build_proxies(cs.xy, cs.start, 10)
    assert st == orc.OK
    assert orc.sort_order(px).tolist() == e["order"]


@pytest.mark.parametrize("name", ["O5_orient_exact_ten_percent", "O6_orient_exact_ten_percent_right"])
def test_orientation_exact_ten_percent(orc, name):
    e = G[name]
    p = _proxy(orc, e["poly"], e["k"])
    assert p.rot90 == 0
    assert (p.fx, p.fy) == (e["fx"], e["fy"])


@pytest.mark.parametrize("name", ["L1_lock_row_one", "L2_lock_row_one_right"])
def test_lock_row_one(orc, name):
    e = G[name]
    a = orc.make_prof([0] * 6, [2] * 6, [0, 0], e["dright_a"])
    b = orc.make_prof([0] * 9, [2] * 9, e["dleft_b"], [9, 9])
    assert orc.offset_raw(a, b) == e["off"]
    assert orc.locks_raw(a, b, e["delta"]) == (e["a_locked"], e["b_locked"])
