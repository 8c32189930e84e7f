"""Oracle hybrid prefix tail (D23-D26; "Performance Optimization").

Pins: t_opt = 0 is bit-identical to the pure sequential path; every
hybrid packing passes the independent raster validator; the reported L2
stretch equals Sander's definition recomputed from the placements (for a
similarity map the per-triangle stretch is 1/s, aggregated as an area-weighted
RMS) and the SPEC worked value sqrt(2.5); the returned
candidate maximises the area-weighted mean final scale exactly.
"""
import math
from fractions import Fraction

import numpy as np
import pytest

import chartgen

U = 256


def _area2(poly):
    q = [(round(float(x) * U), round(float(y) * U)) for x, y in poly]
    return abs(sum(q[i][0] * q[(i + 1) % len(q)][1] - q[(i + 1) % len(q)][0] * q[i][1]
                   for i in range(len(q))))


def l2_stretch_from_placements(areas, scales):
    """Sander et al. L2 stretch of the packed->input map for per-chart
    similarities: sqrt(sum A_c / s_c^2 / sum A_c)."""
    num = sum(Fraction(a) / (Fraction(s) ** 2) for a, s in zip(areas, scales))
    return math.sqrt(num / sum(Fraction(a) for a in areas))


def test_stretch_helper_spec_example():
    # two equal-area charts at scales 1 and 1/2 -> sqrt((1 + 4)/2)
    assert l2_stretch_from_placements([10, 10], [1, Fraction(1, 2)]) == pytest.approx(
        math.sqrt(2.5), rel=1e-15)


HYB = [chartgen.small_case(s, n=400, family="tss", side=512, rho=0.6) for s in range(2)] + \
      [chartgen.small_case(s, n=300, family="lightmap", side=384, rho=0.9) for s in range(2)]


@pytest.mark.parametrize("cs", HYB, ids=lambda c: c.name)
def test_t_opt_zero_is_sequential(orc, cs):
    a = orc.pack(cs, t_opt_bp=0)
    b = orc.pack(cs, t_opt_bp=-1)  # policy: 0 for <= 10,000 charts
    assert a[0] == b[0] and np.array_equal(a[1], b[1])
    assert a[2].prefix_rows == 0 and set(a[1]["mode"].tolist()) == {0}


@pytest.mark.parametrize("t", [100, 300, 1000])
@pytest.mark.parametrize("cs", HYB, ids=lambda c: c.name)
def test_hybrid_valid_and_stretch(orc, cs, t):
    st, pl, info, cands = orc.pack(cs, t_opt_bp=t, with_cands=True)
    assert st == orc.OK
    assert orc.validate(cs, pl) == {"overlap": 0, "gutter": 0, "oob": 0}
    areas = [_area2(cs.polygon(c)) for c in range(cs.n_charts)]
    scales = [Fraction(int(p["scale_num"]), int(p["scale_den"])) for p in pl]
    assert info.l2_stretch == pytest.approx(l2_stretch_from_placements(areas, scales), rel=1e-12)
    assert info.l2_stretch >= 1.0
    # D25: exact maximiser of A_seq*m*2^20 + A_pre*p*M over successful candidates
    st_, px, _ = orc.build_proxies(cs.xy, cs.start, cs.local_aabb_count)
    perm = orc.sort_order(px)
    apre = np.concatenate([[0], np.cumsum([px[i].area2 for i in perm], dtype=object)])
    M = cs.scale_count
    best, bestV = 0, -1
    for m in range(1, M + 1):
        c = cands[m - 1]
        if not c.success:
            continue
        r0 = c.switched_at if c.switched_at >= 0 else cs.n_charts
        V = apre[r0] * m * 2 ** 20 + (apre[-1] - apre[r0]) * c.p * M
        if V >= bestV:
            best, bestV = m, V
    assert info.scale_index == best
    if info.prefix_rows:
        assert set(pl["mode"].tolist()) == {0, 1} or set(pl["mode"].tolist()) == {1}
        tail = pl[pl["mode"] == 1]
        assert np.all(tail["scale_den"] == 2 ** 20)
        # intermediate DOWNscaling: sigma <= 1 (reading R3)
        assert np.all(tail["scale_num"].astype(np.int64) * M <= best * 2 ** 20)


def test_hybrid_switch_rule(orc):
    """D23: t_opt 1 % of H = 1024 switches once the tallest remaining
    chart is below 10.24 texels (8 texels here); with t_opt = 0 it never does."""
    # a 100-tall chart (no knee: the drop 92 < 10 % of H) then 200 8x8 squares;
    # the first row holds the tall chart and ~100 squares, the second row's
    # tallest chart is 8 < 10.24 texels -> switch there
    polys = [[(0, 0), (40, 0), (40, 100), (0, 100)]] + \
            [[(0, 0), (8, 0), (8, 8), (0, 8)] for _ in range(200)]
    polys = [[(x + 3 * i, y) for x, y in p] for i, p in enumerate(polys)]
    cs = chartgen.from_polygons(polys, 1024, 1024)
    st, pl, info, cands = orc.pack(cs, t_opt_bp=100, with_cands=True)
    assert st == orc.OK and info.prefix_rows >= 1 and info.rows == 1
    assert 1 < cands[info.scale_index - 1].switched_at < 201
    assert orc.validate(cs, pl) == {"overlap": 0, "gutter": 0, "oob": 0}
    st0, pl0, info0, _ = orc.pack(cs, t_opt_bp=0, with_cands=True)
    assert info0.prefix_rows == 0


def test_area_bound_does_not_hold_with_a_prefix_tail(orc):
    """Reading R2 prunes candidates whose scaled total area exceeds
    the atlas -- exact in sequential mode only.  With a hybrid tail the prefix
    rows are downscaled by sigma < 1 (D24), so a candidate above the
    bound can succeed and win (D25): here m = 63 and 64 lie above it and 64 is
    the oracle's winner (found by the random parity sweep; the CUDA path now
    starts its hybrid search at M)."""
    import importlib.util
    import os
    spec = importlib.util.spec_from_file_location(
        "fz", os.path.join(os.path.dirname(__file__), "test_gpu_fuzz.py"))
    fz = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(fz)
    cs, kw = fz.case(105)
    st, pl, info, cands = orc.pack(cs, with_cands=True, **kw)
    a2 = sum(_area2(cs.polygon(c)) for c in range(cs.n_charts))
    M = kw["scale_count"]
    above = [m for m in range(1, M + 1) if m * m * a2 > 2 * 65536 * cs.atlas_w * cs.atlas_h * M * M]
    assert above and info.scale_index in above and cands[info.scale_index - 1].success
    assert cands[info.scale_index - 1].switched_at >= 0 and cands[info.scale_index - 1].p < (1 << 20)
    assert orc.validate(cs, pl) == {"overlap": 0, "gutter": 0, "oob": 0}
