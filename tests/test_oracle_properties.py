"""Oracle pinned to invariants, closed forms and the LOCK-1 counterexample.

* validity ("strictly satisfies the specified gutter sizes"):
  the independent exact raster validator reports zero overlap / gutter / OOB
  texels on every packing of a seeded corpus;
* closed forms: single chart m = max{m : ceil(w m/M) <= W, ceil(h m/M) <= H}
  (S:424), trivial fit -> m = M, stretch = M/m for a uniform scale;
* footprints contain the exact raster coverage (D11 "TopEdge rounded up ...
  BottomEdge rounded down" so that "charts are strictly separated");
* exhaustive-search consistency, determinism;
* D8 mirror self-test; OBB containment/optimality over the 8 angles;
* LOCK-1: the paper-literal adjacent-only Alg. 1 overlaps,
  the D15 extension does not.
"""
import math
from fractions import Fraction

import numpy as np
import pytest

import chartgen

U = 256


def corpus():
    out = []
    out += [chartgen.config1a(s) for s in range(12)]
    out += [chartgen.config1b(s) for s in range(12)]
    out += [chartgen.small_case(s, n=40) for s in range(6)]
    out += [chartgen.small_case(s, n=40, family="uv") for s in range(6)]
    out += [chartgen.small_case(s, n=30, family="mixed", rho=0.9) for s in range(4)]
    return out


@pytest.mark.parametrize("cs", corpus(), ids=lambda c: c.name)
def test_validity_and_search_consistency(orc, cs):
    st, pl, info, cands = orc.pack(cs, with_cands=True)
    assert st == orc.OK
    v = orc.validate(cs, pl)
    assert v == {"overlap": 0, "gutter": 0, "oob": 0}
    succ = [i + 1 for i, c in enumerate(cands) if c.success]
    assert info.scale_index == max(succ)
    assert info.l2_stretch == pytest.approx(64 / info.scale_index, rel=1e-15)
    assert info.l2_stretch >= 1.0
    # every placement is at the chosen uniform scale
    assert set(pl["scale_num"].tolist()) == {info.scale_index}


@pytest.mark.parametrize("cs", corpus()[::3], ids=lambda c: c.name)
def test_area_bound_prunes_only_failures(orc, cs):
    """The CUDA path skips candidates whose scaled total chart area exceeds the
    atlas (DESIGN.md scale search).  That is exact: every such candidate fails in
    the exhaustive oracle, because successful packings are overlap-free and in
    bounds (validator)."""
    st, pl, info, cands = orc.pack(cs, with_cands=True)
    a2 = 0
    for c in range(cs.n_charts):
        q = _snapped(cs.polygon(c))
        a2 += abs(sum(q[i][0] * q[(i + 1) % len(q)][1] - q[(i + 1) % len(q)][0] * q[i][1]
                      for i in range(len(q))))
    M = cs.scale_count
    for m in range(1, M + 1):
        if m * m * a2 > 2 * 65536 * cs.atlas_w * cs.atlas_h * M * M:
            assert not cands[m - 1].success, m


def test_determinism(orc):
    cs = chartgen.small_case(3, n=60, family="uv")
    a = orc.pack(cs)
    b = orc.pack(cs)
    assert a[0] == b[0] and np.array_equal(a[1], b[1]) and a[2].scale_index == b[2].scale_index


def _snapped(poly):
    return [(round(float(x) * U), round(float(y) * U)) for x, y in poly]


@pytest.mark.parametrize("seed", range(20))
def test_single_chart_closed_form(orc, seed):
    rng = chartgen.SplitMix64(seed)
    W = rng.randint(20, 120)
    H = rng.randint(20, 120)
    cs1 = chartgen.generate("mixed", 1, W, H, seed, rho=None)
    scale = rng.uniform(0.5, 4.0)
    poly = [(x * scale, y * scale) for x, y in cs1.polygon(0)]
    cs = chartgen.from_polygons([poly], W, H, gutter=rng.randint(0, 2))
    q = _snapped(cs.polygon(0))
    ex = max(p[0] for p in q) - min(p[0] for p in q)
    ey = max(p[1] for p in q) - min(p[1] for p in q)
    w, h = min(ex, ey), max(ex, ey)  # 90-degree normalization
    M = 64
    ok = [m for m in range(1, M + 1)
          if math.ceil(Fraction(w * m, M * U)) <= W and math.ceil(Fraction(h * m, M * U)) <= H]
    st, pl, info, _ = orc.pack(cs)
    if not ok:
        assert st == orc.NO_FIT
    else:
        assert st == orc.OK and info.scale_index == max(ok)
        assert orc.validate(cs, pl) == {"overlap": 0, "gutter": 0, "oob": 0}


@pytest.mark.parametrize("seed", range(10))
def test_trivial_fit(orc, seed):
    """Sum of dilated widths fits W' and the tallest fits H' => m = M, stretch 1."""
    cs0 = chartgen.generate("mixed", 12, 256, 256, seed, rho=None)
    g = 1
    wd, hd = [], []
    for c in range(cs0.n_charts):
        q = _snapped(cs0.polygon(c))
        ex = max(p[0] for p in q) - min(p[0] for p in q)
        ey = max(p[1] for p in q) - min(p[1] for p in q)
        wd.append(math.ceil(Fraction(min(ex, ey), U)) + 2 * g)
        hd.append(math.ceil(Fraction(max(ex, ey), U)) + 2 * g)
    W = sum(wd) - 2 * g
    H = max(hd) - 2 * g
    cs = chartgen.ChartSet("trivial", cs0.xy, cs0.start, W, H, gutter=g)
    st, pl, info, _ = orc.pack(cs)
    assert st == orc.OK and info.scale_index == 64 and info.l2_stretch == 1.0
    assert orc.validate(cs, pl) == {"overlap": 0, "gutter": 0, "oob": 0}


def _placement(orc, m, M, box_w, box_h, mirror=0):
    p = np.zeros(1, dtype=orc.PLACEMENT_DTYPE)[0]
    p["scale_num"], p["scale_den"], p["box_w"], p["box_h"], p["mirror_x"] = m, M, box_w, box_h, mirror
    return p


@pytest.mark.parametrize("k", [1, 2, 5, 10, 17])
def test_footprint_contains_raster_coverage(orc, k):
    """Every texel whose open square meets the chart lies inside its footprint
    (columns: Top <= r < Bot; rows: Left <= i < Right), also mirrored."""
    sets = [chartgen.config1a(1), chartgen.small_case(2, n=30, family="uv", side=512)]
    for cs in sets:
        st, px, _ = orc.build_proxies(cs.xy, cs.start, k)
        assert st == orc.OK
        for c in range(cs.n_charts):
            p = px[c]
            for m in (64, 47, 23, 5):
                pr = orc.Profile(p, m, 64, 0)
                for mirror in (0, 1):
                    pl = _placement(orc, m, 64, pr.ws, pr.hs, mirror)
                    pl["rot90"], pl["flip_x"], pl["flip_y"] = p.rot90, p.fx, p.fy
                    mask = orc.raster_chart(cs.polygon(c), pl, 0, 0, pr.ws, pr.hs)
                    top = pr.Dtop[::-1] if mirror else pr.Dtop
                    bot = pr.Dbot[::-1] if mirror else pr.Dbot
                    rows, cols = np.nonzero(mask)
                    assert np.all(rows >= top[cols]) and np.all(rows < bot[cols])
                    if not mirror:
                        assert np.all(cols >= pr.Dleft[rows]) and np.all(cols < pr.Dright[rows])
                    # coverage reaches every column and row of the box (D12)
                    assert mask.any(axis=0).all() and mask.any(axis=1).all()


def test_dilation_is_chebyshev(orc):
    cs = chartgen.config1a(4)
    st, px, _ = orc.build_proxies(cs.xy, cs.start, 10)
    for c in range(cs.n_charts):
        p0 = orc.Profile(px[c], 37, 64, 0)
        for g in (1, 2):
            pg = orc.Profile(px[c], 37, 64, g)
            assert pg.Wd == p0.Wd + 2 * g and pg.Hd == p0.Hd + 2 * g
            for i in range(pg.Wd):
                lo, hi = max(0, i - 2 * g), min(i, p0.Wd - 1)
                assert pg.Dtop[i] == p0.Dtop[lo:hi + 1].min()
                assert pg.Dbot[i] == p0.Dbot[lo:hi + 1].max() + 2 * g


def _posed(orc, cs, c, p):
    q = _snapped(cs.polygon(c))
    xmin = min(v[0] for v in q)
    ymin = min(v[1] for v in q)
    pts = [(x - xmin, y - ymin) for x, y in q]
    if p.rot90:
        pts = [(p.w - y, x) for x, y in pts]
    if p.fx:
        pts = [(p.w - x, y) for x, y in pts]
    if p.fy:
        pts = [(x, p.h - y) for x, y in pts]
    return pts


def test_obb_containment_and_optimality(orc):
    cs = chartgen.generate("tss", 200, 1024, 1024, 9, rho=0.5)
    st, px, _ = orc.build_proxies(cs.xy, cs.start, 10)
    src = open(orc.HERE + "/tabi_oracle.c").read()
    import re
    QC = [int(v) for v in re.search(r"OR_QC\[8\] = \{([^}]*)\}", src).group(1).split(",")]
    QS = [int(v) for v in re.search(r"OR_QS\[8\] = \{([^}]*)\}", src).group(1).split(",")]
    for c in range(cs.n_charts):
        p = px[c]
        pts = _posed(orc, cs, c, p)
        assert min(x for x, _ in pts) == 0 and max(x for x, _ in pts) == p.w
        assert min(y for _, y in pts) == 0 and max(y for _, y in pts) == p.h
        areas = []
        for j in range(8):
            u = [x * QC[j] + y * QS[j] for x, y in pts]
            v = [-x * QS[j] + y * QC[j] for x, y in pts]
            areas.append((max(u) - min(u)) * (max(v) - min(v)))
        assert areas[p.obb_j] == min(areas)
        assert p.obb_j == areas.index(min(areas))
        j = p.obb_j
        for x, y in pts:
            assert p.umin <= x * QC[j] + y * QS[j] <= p.umax
            assert p.vmin <= -x * QS[j] + y * QC[j] <= p.vmax


def test_mirror_self_consistency(orc):
    """D8: a chart and its mirror image end in the same final pose unless the
    orientation rule ties (then neither is reflected)."""
    cs = chartgen.generate("uv", 80, 512, 512, 5, rho=0.7)
    st, px, _ = orc.build_proxies(cs.xy, cs.start, 10)
    polys = []
    for c in range(cs.n_charts):
        poly = cs.polygon(c).astype(np.float64)
        if px[c].rot90:  # posed x is input -y
            poly = np.stack([poly[:, 0], -poly[:, 1]], 1)
        else:
            poly = np.stack([-poly[:, 0], poly[:, 1]], 1)
        polys.append(poly[::-1] + 2048.0)
    mcs = chartgen.from_polygons(polys, 512, 512)
    st, qx, _ = orc.build_proxies(mcs.xy, mcs.start, 10)
    same = 0
    for p, q in zip(px, qx):
        if p.fx != q.fx:
            fields = ("w", "h", "fy", "obb_j", "umin", "umax", "vmin", "vmax")
            assert all(getattr(p, f) == getattr(q, f) for f in fields)
            assert list(p.top) == list(q.top) and list(p.bot) == list(q.bot)
            assert list(p.left) == list(q.left) and list(p.right) == list(q.right)
            same += 1
        else:
            assert p.fx == 0 and q.fx == 0
    assert same >= 60


def test_nested_k_tightness(orc):
    """Local-AABB proxy area shrinks as the partition refines when k | k'
    (SPEC S:186 claims it for 2 vs 5 too, which does not hold in general)."""
    cs = chartgen.generate("uv", 120, 1024, 1024, 2, rho=0.8)
    areas = {}
    for k in (1, 5, 10, 20):
        st, px, _ = orc.build_proxies(cs.xy, cs.start, k)
        areas[k] = [Fraction(sum(p.bot[j] - p.top[j] for j in range(k)) * p.w, k) for p in px]
    for c in range(cs.n_charts):
        assert areas[20][c] <= areas[10][c] <= areas[5][c] <= areas[1][c]


def _lock1(orc, flags):
    """SURVEY Appendix C with the arm moved from y in [40, 42] to [45, 47]: with
    k = 10 the closed y-slice [30, 40] would otherwise see the arm's top edge and
    forbid the compaction the counterexample needs (readings)."""
    A = [(0, 0), (20, 0), (20, 150), (0, 150)]
    c0 = [(0, 0), (10, 0), (10, 45), (40, 45), (40, 47), (10, 47), (10, 100), (0, 100)]
    c1 = [(0, 0), (10, 0), (10, 35), (0, 35)]
    c2 = [(0, 0), (10, 0), (10, 30), (0, 30)]
    cs = chartgen.from_polygons([A, c0, c1, c2], 40, 256, gutter=0)
    st, pl, info, _ = orc.pack(cs, flags=flags)
    return cs, st, pl, info


def test_lock1_literal_adjacent_locks_overlap(orc):
    cs, st, pl, info = _lock1(orc, orc.F_ADJACENT_LOCKS_ONLY)
    assert st == orc.OK and info.scale_index == 64
    # the arm (rows 150-151 over columns 0-27) meets c2 (columns 10-19): 20 texels
    assert orc.validate(cs, pl)["overlap"] == 20


def test_lock1_extended_locks_no_overlap(orc):
    cs, st, pl, info = _lock1(orc, 0)
    assert st == orc.OK and info.scale_index == 64
    assert orc.validate(cs, pl) == {"overlap": 0, "gutter": 0, "oob": 0}


def test_invalid_inputs(orc):
    cs = chartgen.from_polygons([[(0, 0), (1, 0), (1, 1)], [(0, 0), (5, 0), (10, 0)]], 64, 64)
    st, _, info, _ = orc.pack(cs)
    assert st == orc.EINVAL and info.bad_chart == 1  # zero area after snapping
    cs = chartgen.from_polygons([[(0, 0), (1, 0)]], 64, 64)
    st, _, info, _ = orc.pack(cs)
    assert st == orc.EINVAL and info.bad_chart == 0  # < 3 vertices
    cs = chartgen.from_polygons([[(0, 0), (1, 0), (float("nan"), 1)]], 64, 64)
    st, _, info, _ = orc.pack(cs)
    assert st == orc.EINVAL and info.bad_chart == 0
    cs = chartgen.from_polygons([[(0, 0), (1, 0), (0, 1)]], 0, 64)
    st, _, _, _ = orc.pack(cs)
    assert st == orc.EINVAL


def test_footprint_extremes_equal_the_dilated_box(orc):
    """Every dilated footprint reaches its box: max_j BottomEdge = Hd,
    min_j TopEdge = 0, max_i Right = Wd, min_i Left = 0 (D11: the footprint
    contains the chart, whose extreme points lie in some column / row, and is
    clipped to the chart extent; D13: the dilation adds 2g).  The CUDA push
    relies on it (the score of a chart is Y + Hd)."""
    cases = [chartgen.small_case(s, n=40, family=f, rho=r)
             for s, (f, r) in enumerate([("uv", 0.8), ("tss", 1.2), ("mixed", 0.5),
                                         ("lightmap", 1.0)])]
    checked = 0
    for cs in cases:
        for k in (1, 3, 10):
            st, px, _ = orc.build_proxies(cs.xy, cs.start, k)
            assert st == orc.OK
            for p in px:
                for num, den, g in ((64, 64, 1), (37, 64, 0), (5, 16, 2), (912345, 1 << 20, 1)):
                    pr = orc.Profile(p, num, den, g)
                    assert max(pr.Dbot) == pr.Hd and min(pr.Dtop) == 0
                    assert max(pr.Dright) == pr.Wd and min(pr.Dleft) == 0
                    checked += 1
    assert checked > 1000


# Polygons symmetric about the diagonal x = y whose minimum-area boxes over
# the 8 angles of D6 are tied between j and 8 - j (the Q30 table has
# C_{8-j} = S_j, so the mirror image ties exactly in integers).
D6_TIES = [[(0, 0), (27, 10), (37, 37), (10, 27)],
           [(0, 0), (14, 9), (23, 23), (9, 14)],
           [(0, 0), (71, 18), (89, 89), (18, 71)],
           [(0, 0), (41, 19), (80, 40), (90, 90), (40, 80), (19, 41)],
           [(0, 0), (33, 23), (66, 46), (105, 63), (112, 112), (63, 105), (46, 66), (23, 33)]]
_QC = [1073741824, 1053110176, 992008094, 892783698, 759250125, 596538995, 410903207, 209476638]
_QS = [0, 209476638, 410903207, 596538995, 759250125, 892783698, 992008094, 1053110176]


def test_obb_angle_tie_takes_the_smaller_angle(orc):
    """D6 tie rule ('ties -> smaller j'): on shapes whose two best
    angles give exactly equal box areas, the oracle's OBB is the smaller j --
    the areas recomputed here from the snapped outline (any reflection of the
    final pose maps j to 8 - j, which the symmetry leaves tied)."""
    for poly in D6_TIES:
        q = [(x * 256, y * 256) for x, y in poly]
        areas = []
        for j in range(8):
            us = [x * _QC[j] + y * _QS[j] for x, y in q]
            vs = [-x * _QS[j] + y * _QC[j] for x, y in q]
            areas.append((max(us) - min(us)) * (max(vs) - min(vs)))
        best = min(areas)
        tied = [j for j in range(8) if areas[j] == best]
        assert len(tied) == 2 and tied[0] + tied[1] == 8 and tied[0] in (1, 2, 3), (poly, tied)
        cs = chartgen.from_polygons([poly], 512, 512)
        st, px, _ = orc.build_proxies(cs.xy, cs.start, 10)
        assert st == orc.OK and px[0].obb_j == tied[0], (poly, px[0].obb_j, tied)
        # and the box is that angle's: its extents give the minimum area
        assert (px[0].umax - px[0].umin) * (px[0].vmax - px[0].vmin) == best
