"""Oracle pinned to hand-derived goldens (tests/golden/goldens.json).

Every expected value is restated from SPEC.md / PAPER.md examples (cited per
case) under this build's integer conventions; none is
produced by the code under test.
"""
import json
import math
import os

import numpy as np
import pytest

import chartgen

G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "goldens.json")))
U = 256  # units per texel (D2)


def _proxy(orc, poly, k):
    cs = chartgen.from_polygons([poly], 64, 64)
    st, px, bad = orc.build_proxies(cs.xy, cs.start, k)
    assert st == orc.OK
    return px[0]


def test_A1_slices_tri_tl(orc):
    p = _proxy(orc, G["tri_tl"]["poly"], 2)
    e = G["A1_xslices_k2"]
    assert (p.w, p.h, p.rot90, p.fx, p.fy) == (8 * U, 8 * U, 0, 0, 0)
    assert list(p.top[:2]) == [v * U for v in e["top"]]
    assert list(p.bot[:2]) == [v * U for v in e["bot"]]
    assert list(p.left[:2]) == [v * U for v in e["left"]]
    assert list(p.right[:2]) == [v * U for v in e["right"]]


def test_A2_A3_column_and_row_profiles(orc):
    p = _proxy(orc, G["tri_tl"]["poly"], 2)
    pr = orc.Profile(p, 64, 64, 0)
    assert pr.Wd == 8 and pr.Hd == 8
    assert pr.Dbot.tolist() == G["A2_bot_columns_k2"]["bot"]
    assert pr.Dtop.tolist() == [0] * 8
    assert pr.Dright.tolist() == G["A3_right_rows_k2"]["right"]
    assert pr.Dleft.tolist() == [0] * 8


def test_A4_A5_offset_and_locks(orc):
    e = G["A4_offset"]
    a = orc.make_prof([0] * 8, [8] * 8, [0] * 8, e["dright_a"])
    b = orc.make_prof([0] * 8, [8] * 8, e["dleft_b"], [8] * 8)
    assert orc.offset_raw(a, b) == e["off"]
    la, lb = orc.locks_raw(a, b, e["off"])
    assert la == G["A5_locks"]["a_locked"] and lb == G["A5_locks"]["b_locked"]


def test_A4_offset_is_conservative_vs_raster(orc):
    """The proxy offset never undercuts the exact raster minimum: Tri-TL
    and Tri-BR both cover the diagonal texels x+y=7, so the raster minimum advance
    is 1 while the k=2 proxy gives 4 >= 1."""
    tl = orc.raster_chart(np.array(G["tri_tl"]["poly"], dtype=np.float32),
                          _ident(), 0, 0, 8, 8)
    br = orc.raster_chart(np.array(G["tri_br"]["poly"], dtype=np.float32),
                          _ident(), 0, 0, 8, 8)
    best = None
    for adv in range(0, 9):
        clash = False
        for y in range(8):
            for x in range(8):
                if tl[y, x] and 0 <= x - adv < 8 and br[y, x - adv]:
                    clash = True
        if not clash:
            best = adv
            break
    assert best == 1
    assert G["A4_offset"]["off"] >= best


def _ident(**kw):
    import oracle
    p = np.zeros(1, dtype=oracle.PLACEMENT_DTYPE)[0]
    p["scale_num"] = 1
    p["scale_den"] = 1
    for k_, v in kw.items():
        p[k_] = v
    return p


def test_A6_orientation(orc):
    p = _proxy(orc, G["tri_tl"]["poly"], 2)
    assert (p.fx, p.fy) == (G["A6_orient_tri_tl"]["fx"], G["A6_orient_tri_tl"]["fy"])
    q = _proxy(orc, G["tri_br"]["poly"], 2)
    assert (q.fx, q.fy) == (G["A6b_orient_tri_br"]["fx"], G["A6b_orient_tri_br"]["fy"])
    # after both reflections Tri-BR is Tri-TL: identical final-pose proxy (D8)
    assert list(q.top[:2]) == list(p.top[:2]) and list(q.bot[:2]) == list(p.bot[:2])


def test_A7_obb(orc):
    p = _proxy(orc, G["tri_tl"]["poly"], 2)
    assert p.obb_j == G["A7_obb_tri_tl"]["obb_j"]


@pytest.mark.parametrize("name", ["A8_fold_nohc", "A9_fold_hc", "A10_fold_first_overflows"])
def test_fold(orc, name):
    e = G[name]
    end, x = orc.fold_row(e["widths"], e["offs"], 0, e["fold_w"], e["hc"])
    assert end == e["end"] and x == e["x"]


@pytest.mark.parametrize("name", ["A11_correct_pair", "A12_correct_chain"])
def test_correct_y(orc, name):
    e = G[name]
    assert orc.correct_y([tuple(p) for p in e["pairs"]], e["y"]) == e["out"]


def test_correct_y_no_locks_unchanged(orc):
    assert orc.correct_y([(0, 1, 0, 0)], [7, 3]) == [7, 3]


@pytest.mark.parametrize("name", ["A13_knee_update", "A14_knee_update_stays", "A14b_knee_collapse"])
def test_knee_update(orc, name):
    e = G[name]
    ok, left, right = orc.update_knee(e["F"], e["ltr"], e["left"], e["right"])
    assert ok == e["ok"]
    if ok:
        assert right == e["new_right"] and left == e["left"]


def test_knee_update_rtl_mirror(orc):
    """Alg. 2's right-to-left branch is the mirror image of A13."""
    ok, left, right = orc.update_knee([3, 2, 2, 10, 10], 0, 1, 5)
    assert ok and (left, right) == (3, 5)


@pytest.mark.parametrize("name", ["A15_knee", "A16_no_knee", "A17_largest_knee"])
def test_find_knee(orc, name):
    e = G[name]
    assert orc.find_knee([h * U for h in e["heights"]], e["atlas_h"]) == e["knee"]


def test_knee_thresholds_inclusive(orc):
    """>= at both thresholds: H=100 -> 10 texels; taller 50 -> 10 texels."""
    assert orc.find_knee([50 * U, 40 * U], 100) == 0
    assert orc.find_knee([50 * U, 40 * U + 1], 100) == -1


def test_A18_push(orc):
    e = G["A18_push"]
    assert orc.push_y(e["F"], 0, e["dtop"]) == e["y"]


@pytest.mark.parametrize("name", ["A19_single_small", "A20_single_big"])
def test_single_chart(orc, name):
    e = G[name]
    cs = chartgen.from_polygons([e["poly"]], e["atlas"], e["atlas"], gutter=e["gutter"])
    st, pl, info, _ = orc.pack(cs)
    assert st == orc.OK
    assert info.scale_index == e["m"]
    assert info.l2_stretch == pytest.approx(e["stretch"], rel=1e-12)
    assert orc.validate(cs, pl) == {"overlap": 0, "gutter": 0, "oob": 0}


def test_A21_no_fit(orc):
    e = G["A21_too_wide"]
    cs = chartgen.from_polygons([e["poly"]], e["atlas"], e["atlas"], gutter=e["gutter"])
    st, _, info, _ = orc.pack(cs)
    assert st == e["status"] == orc.NO_FIT
    assert info.scale_index == 0


def test_A24_validator_gutter(orc):
    sq = [[0, 0], [1, 0], [1, 1], [0, 1]]
    cs = chartgen.from_polygons([sq, sq], 8, 8, gutter=1)
    pl = np.zeros(2, dtype=orc.PLACEMENT_DTYPE)
    for i, tx in enumerate((0, 2)):
        pl[i] = _ident(tx=tx, box_w=1, box_h=1)
    # texels (1,0) and (1,1) lie in both 1-px Chebyshev dilations
    assert orc.validate(cs, pl) == {"overlap": 0, "gutter": 2, "oob": 0}
    pl[1]["tx"] = 3
    assert orc.validate(cs, pl) == {"overlap": 0, "gutter": 0, "oob": 0}
    pl[1]["tx"] = 0
    assert orc.validate(cs, pl)["overlap"] == 1
    pl[1]["tx"] = 8
    assert orc.validate(cs, pl)["oob"] == 1


def test_q30_table_against_libm():
    """Appendix B's Q30 table is round(cos/sin(j*pi/16) * 2^30)."""
    src = open(os.path.join(os.path.dirname(__file__), "..", "oracle", "tabi_oracle.c")).read()
    import re
    qc = [int(v) for v in re.search(r"OR_QC\[8\] = \{([^}]*)\}", src).group(1).replace("\n", "").split(",")]
    qs = [int(v) for v in re.search(r"OR_QS\[8\] = \{([^}]*)\}", src).group(1).replace("\n", "").split(",")]
    for j in range(8):
        assert abs(qc[j] - math.cos(j * math.pi / 16) * 2 ** 30) <= 0.5
        assert abs(qs[j] - math.sin(j * math.pi / 16) * 2 ** 30) <= 0.5
