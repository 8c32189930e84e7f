"""Oracle pins for R4 pre-rotation (TABI_F_PREROTATE).

P:1022 "We pre-rotate the UV charts to align their tight bounding boxes with
the major axes prior to packing"; S:408-416 rotate "by the negative of its
approximate-OBB angle".  DESIGN.md R4: the angle is D6's minimum-area angle
over j*pi/16, j = 0..7, of the snapped polygon; the rotated coordinates are
rounded half to even to 1/256 texel; placements carry the index (step 0 of
tabi_placement) and the validator applies it to the ORIGINAL outline.

Pins independent of the oracle's own arithmetic:
* the chosen angle is the float argmin of the rotated-AABB area computed with
  math.cos/sin (not the Q30 table), away from near-ties;
* a rectangle rotated by j*pi/16 comes back as the axis-aligned rectangle:
  prerot = j (mod the 90-degree symmetry) and w*h = a*b within rounding;
* flags=0 and axis-aligned input are untouched (prerot 0, identical proxies);
* every pre-rotated packing of a seeded corpus is valid under the raster
  validator, which rasterizes the original polygons through step 0;
* on rotated rectangles pre-rotation packs at a scale no worse than without.
"""
import math

import numpy as np
import pytest

import chartgen

U = 256.0


def _proxy_fields(p):
    return (p.w, p.h, p.area2, p.xmin, p.ymin, p.rot90, p.fx, p.fy, p.obb_j,
            tuple(p.top), tuple(p.bot), tuple(p.left), tuple(p.right),
            p.umin, p.umax, p.vmin, p.vmax)


def _chartset(polys, W=256, H=256, name="pr"):
    xy, start = [], [0]
    for p in polys:
        for (x, y) in p:
            xy += [round(x * U) / U, round(y * U) / U]
        start.append(start[-1] + len(p))
    return chartgen.ChartSet(name=name, xy=np.asarray(xy, dtype=np.float32),
                             start=np.asarray(start, dtype=np.int32), atlas_w=W, atlas_h=H)


def _rot(pts, th, ox=100.0, oy=90.0):
    c, s = math.cos(th), math.sin(th)
    return [(ox + x * c - y * s, oy + x * s + y * c) for (x, y) in pts]


def _rect(a, b):
    return [(-a / 2, -b / 2), (a / 2, -b / 2), (a / 2, b / 2), (-a / 2, b / 2)]


def _float_areas(poly):
    """Rotated-AABB area of the snapped polygon in the frame
    (u, v) = (x cos + y sin, -x sin + y cos), for theta = j pi / 16."""
    q = [(round(x * U), round(y * U)) for (x, y) in poly]
    out = []
    for j in range(8):
        c, s = math.cos(j * math.pi / 16), math.sin(j * math.pi / 16)
        us = [x * c + y * s for (x, y) in q]
        vs = [-x * s + y * c for (x, y) in q]
        out.append((max(us) - min(us)) * (max(vs) - min(vs)))
    return out


def test_flag_off_and_axis_aligned_untouched(orc):
    for seed in range(4):
        cs = chartgen.config1b(seed)  # rectangles and L-shapes, axis-aligned
        st0, p0, _ = orc.build_proxies(cs.xy, cs.start, 10)
        st1, p1, _ = orc.build_proxies(cs.xy, cs.start, 10, flags=orc.F_PREROTATE)
        assert st0 == st1 == orc.OK
        for a, b in zip(p0, p1):
            assert a.prerot == 0 and b.prerot == 0
            assert _proxy_fields(a) == _proxy_fields(b)
    cs = chartgen.config1a(0)
    st, p0, _ = orc.build_proxies(cs.xy, cs.start, 10)
    assert all(p.prerot == 0 for p in p0)


@pytest.mark.parametrize("j", range(1, 8))
def test_rotated_rectangle_is_straightened(orc, j):
    a, b = 120.0, 30.0
    cs = _chartset([_rot(_rect(a, b), j * math.pi / 16)])
    st, px, _ = orc.build_proxies(cs.xy, cs.start, 10, flags=orc.F_PREROTATE)
    assert st == orc.OK
    p = px[0]
    assert p.prerot == j
    # the AABB of the straightened chart is the rectangle up to the 1/256 snap
    # of the input and the 1/256 rounding of the rotation (a few units each)
    assert abs(max(p.w, p.h) - a * U) <= 4 and abs(min(p.w, p.h) - b * U) <= 4
    # and its area equals the polygon area (a rectangle fills its box)
    assert abs(p.w * p.h - p.area2 / 2) <= 4 * (a + b) * U


@pytest.mark.parametrize("seed", range(6))
def test_angle_is_float_argmin(orc, seed):
    cs = chartgen.generate("tss", 40, 512, 512, seed, rho=None)
    st, px, _ = orc.build_proxies(cs.xy, cs.start, 10, flags=orc.F_PREROTATE)
    assert st == orc.OK
    checked = 0
    for c in range(cs.n_charts):
        ar = _float_areas(cs.polygon(c))
        best = min(ar)
        srt = sorted(ar)
        if srt[1] - srt[0] <= 1e-9 * best + 1e3:  # near-tie: Q30 rounding may decide
            continue
        assert px[c].prerot == ar.index(best), (c, ar)
        checked += 1
    assert checked >= 30


def _pre_corpus():
    out = [chartgen.small_case(s, n=40, family="uv") for s in range(4)]
    out += [chartgen.generate("tss", 60, 256, 256, s, rho=0.5, name=f"tss-{s}") for s in range(4)]
    out += [chartgen.generate("mixed", 30, 256, 256, s, rho=0.6, name=f"mix-{s}") for s in range(3)]
    return out


@pytest.mark.parametrize("cs", _pre_corpus(), ids=lambda c: c.name)
def test_prerotated_packings_are_valid(orc, cs):
    st, pl, info, cands = orc.pack(cs, with_cands=True, flags=orc.F_PREROTATE)
    assert st == orc.OK
    assert orc.validate(cs, pl) == {"overlap": 0, "gutter": 0, "oob": 0}
    succ = [i + 1 for i, c in enumerate(cands) if c.success]
    assert info.scale_index == max(succ)
    _, px, _ = orc.build_proxies(cs.xy, cs.start, cs.local_aabb_count, flags=orc.F_PREROTATE)
    assert pl["prerot"].tolist() == [p.prerot for p in px]


def test_validator_sees_prerotation(orc):
    """Dropping step 0 from a pre-rotated placement must be caught: the
    validator rasterizes the original outline, so a placement whose box was
    computed for the straightened chart no longer covers it."""
    polys = [_rot(_rect(100, 12), 4 * math.pi / 16, 60, 60),
             _rot(_rect(100, 12), 4 * math.pi / 16, 160, 160)]
    cs = _chartset(polys)
    st, pl, info, _ = orc.pack(cs, with_cands=True, flags=orc.F_PREROTATE)
    assert st == orc.OK
    assert (pl["prerot"] == 4).all()
    assert orc.validate(cs, pl) == {"overlap": 0, "gutter": 0, "oob": 0}
    bad = pl.copy()
    bad["prerot"] = 0
    v = orc.validate(cs, bad)
    assert v["overlap"] + v["gutter"] + v["oob"] > 0


def test_prerotation_improves_rotated_rectangles(orc):
    rng = chartgen.SplitMix64(7)
    polys = []
    for i in range(24):
        a, b = rng.uniform(20, 60), rng.uniform(6, 14)
        j = rng.randint(1, 7)
        polys.append(_rot(_rect(a, b), j * math.pi / 16, rng.uniform(0, 200), rng.uniform(0, 200)))
    cs = _chartset(polys, 112, 112)  # measured: m = 42 without, 58 with
    st0, _, i0, _ = orc.pack(cs, with_cands=True)
    st1, pl1, i1, _ = orc.pack(cs, with_cands=True, flags=orc.F_PREROTATE)
    assert st0 == st1 == orc.OK
    assert i1.scale_index > i0.scale_index
    assert i1.l2_stretch < i0.l2_stretch
    assert orc.validate(cs, pl1) == {"overlap": 0, "gutter": 0, "oob": 0}
