"""Oracle pins for the validator counts and atlas metrics.

Closed forms of the conservative raster rule (texel (i, r) covered
iff the open square (i, i+1) x (r, r+1) meets the closed outline):
* an a x b axis-aligned rectangle at integer offset covers exactly a*b texels,
  and after a g-dilation a*b grows to (a+2g)(b+2g);
* the right triangle (0,0),(8,0),(0,8) covers the 36 texels with i + r <= 7;
* two unit-gap rectangles overlap nowhere, but their g = 1 dilations meet on
  the gap column; a pair shifted onto each other overlaps by the shared area;
* charts hanging over the atlas edge count their outside texels as oob;
* the L2 stretch of a uniform-scale packing is M/m, and equals
  the packer's own figure for hybrid packings (area-weighted RMS, D26).
"""
import numpy as np
import pytest

import chartgen


def _cs(polys, W=64, H=64, g=1):
    xy, start = [], [0]
    for p in polys:
        for (x, y) in p:
            xy += [x, y]
        start.append(start[-1] + len(p))
    return chartgen.ChartSet(name="m", xy=np.asarray(xy, dtype=np.float32),
                             start=np.asarray(start, dtype=np.int32), atlas_w=W, atlas_h=H,
                             gutter=g)


def _pl(orc, rows):
    """rows: (tx, ty, box_w, box_h[, num, den]) with the identity pose."""
    out = np.zeros(len(rows), dtype=orc.PLACEMENT_DTYPE)
    for i, r in enumerate(rows):
        out[i]["tx"], out[i]["ty"], out[i]["box_w"], out[i]["box_h"] = r[:4]
        out[i]["scale_num"], out[i]["scale_den"] = (r[4], r[5]) if len(r) > 4 else (1, 1)
    return out


def _rect(a, b, x=0.0, y=0.0):
    return [(x, y), (x + a, y), (x + a, y + b), (x, y + b)]


@pytest.mark.parametrize("a,b,g", [(5, 3, 0), (5, 3, 1), (7, 11, 2), (1, 1, 3)])
def test_rectangle_coverage_closed_form(orc, a, b, g):
    cs = _cs([_rect(a, b, 100.0, 200.0)], g=g)  # pose translates the AABB to the origin
    m = orc.metrics(cs, _pl(orc, [(10, 20, a, b)]))
    assert m["covered"] == a * b
    assert m["overlap"] == m["gutter"] == m["oob"] == 0
    assert m["occupancy"] == a * b / (64 * 64)
    assert m["l2_stretch"] == 1.0


def test_triangle_coverage_closed_form(orc):
    cs = _cs([[(0, 0), (8, 0), (0, 8)]])
    m = orc.metrics(cs, _pl(orc, [(3, 4, 8, 8)]))
    assert m["covered"] == 36  # texels with i + r <= 7
    # at scale 1/2 the triangle has legs 4: i + r <= 3 -> 10 texels; stretch 2
    m = orc.metrics(cs, _pl(orc, [(3, 4, 4, 4, 1, 2)]))
    assert m["covered"] == 10
    assert m["l2_stretch"] == 2.0


def test_gutter_and_overlap_closed_forms(orc):
    cs = _cs([_rect(4, 6), _rect(4, 6)])
    # one-texel gap: no overlap, dilations (g = 1) meet on the gap column
    m = orc.metrics(cs, _pl(orc, [(10, 10, 4, 6), (15, 10, 4, 6)]))
    assert m["overlap"] == 0 and m["gutter"] == 6 + 2
    # two-texel gap: clear
    m = orc.metrics(cs, _pl(orc, [(10, 10, 4, 6), (16, 10, 4, 6)]))
    assert m["overlap"] == 0 and m["gutter"] == 0
    # shifted by (2, 3): shared area 2 x 3
    m = orc.metrics(cs, _pl(orc, [(10, 10, 4, 6), (12, 13, 4, 6)]))
    assert m["overlap"] == 6
    assert m["covered"] == 2 * 24 - 6
    # dilated boxes 6 x 8 shifted by (2, 3) share 4 x 5
    assert m["gutter"] == 20


def test_oob_closed_form(orc):
    cs = _cs([_rect(4, 6)], W=32, H=32)
    m = orc.metrics(cs, _pl(orc, [(30, -2, 4, 6)]))
    # columns 30..33 x rows -2..3: inside = 2 x 4
    assert m["oob"] == 24 - 8 and m["covered"] == 8


def test_stretch_matches_packer(orc):
    for cs in [chartgen.config2(0), chartgen.small_case(1, n=60, family="uv")]:
        st, pl, info, _ = orc.pack(cs, with_cands=True)
        m = orc.metrics(cs, pl)
        assert m["l2_stretch"] == pytest.approx(cs.scale_count / info.scale_index, rel=1e-15)
        assert m["overlap"] == m["gutter"] == m["oob"] == 0
        assert 0 < m["occupancy"] < 1
    cs = chartgen.small_case(0, n=400, family="tss", side=512, rho=0.6)
    st, pl, info, _ = orc.pack(cs, with_cands=True, t_opt_bp=300)
    assert info.prefix_rows > 0
    m = orc.metrics(cs, pl)
    assert m["l2_stretch"] == pytest.approx(info.l2_stretch, rel=1e-12)
