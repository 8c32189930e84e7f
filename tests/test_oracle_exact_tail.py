"""Oracle pins for the exact-greedy hybrid tail (TABI_F_EXACT_TAIL; SURVEY
§8(f) N4; reading R6).

R6 keeps D23's switch and D24's row placement (FastAtlas alternation, pushed
with locks, no knees) but folds the tail exactly by Alg. 3 with compaction
(HC on as in the tail) at the candidate scale m/M, so no
row overflows and there is no intermediate downscale.

Pins:
* closed form on N equal a x a squares switched at row 0 (t_opt = 100 %):
  rows of K = floor(W' / (ceil(a m / M) + 2g)) squares stacked with pitch
  ceil(a m / M) + 2g, so m* = max{m : ceil(N / K) * pitch <= H'} -- and the
  sequential path (t_opt = 0) reaches the same m*, while D24's prefix fold
  overflows rows and downscales;
* every chart keeps scale m/M (tail charts mode 1), stretch = M/m exactly;
* packings valid under the raster validator;
* measured claim (SURVEY N4 "likely better stretch than D24"): never worse
  than D24 on the seeded hybrid corpus, strictly better on some.
"""
import numpy as np
import pytest

import chartgen


def _squares(N, a, W=64, H=64, seed=0):
    rng = np.random.default_rng(seed)
    xy, start = [], [0]
    for _ in range(N):
        x0, y0 = int(rng.integers(0, 200)), int(rng.integers(0, 200))
        xy += [x0, y0, x0 + a, y0, x0 + a, y0 + a, x0, y0 + a]
        start.append(start[-1] + 4)
    return chartgen.ChartSet(name=f"sq{N}x{a}", xy=np.asarray(xy, dtype=np.float32),
                             start=np.asarray(start, dtype=np.int32), atlas_w=W, atlas_h=H)


def _m_star(N, a, W, H, g=1, M=64):
    best = 0
    for m in range(1, M + 1):
        pitch = -(-a * m // M) + 2 * g
        K = (W + 2 * g) // pitch
        if K >= 1 and -(-N // K) * pitch <= H + 2 * g:
            best = m
    return best


@pytest.mark.parametrize("N,a", [(37, 10), (50, 7), (20, 13), (1, 30), (64, 8)])
def test_squares_closed_form(orc, N, a):
    cs = _squares(N, a, seed=N)
    m_star = _m_star(N, a, cs.atlas_w, cs.atlas_h)
    st, pl, info, _ = orc.pack(cs, with_cands=True, t_opt_bp=10000, flags=orc.F_EXACT_TAIL)
    assert st == orc.OK
    assert info.scale_index == m_star
    assert info.l2_stretch == cs.scale_count / m_star
    assert (pl["mode"] == 1).all()  # switched at row 0: every chart is in the tail
    assert (pl["scale_num"] == m_star).all() and (pl["scale_den"] == cs.scale_count).all()
    assert orc.validate(cs, pl) == {"overlap": 0, "gutter": 0, "oob": 0}
    st, _, info0, _ = orc.pack(cs, with_cands=True)  # sequential path
    assert info0.scale_index == m_star


def test_prefix_tail_differs_on_squares(orc):
    """The pin discriminates: D24's prefix fold lets the last chart of a row
    overflow and rescales the tail (p / 2^20 < m / M)."""
    cs = _squares(37, 10, seed=37)
    st, pl, info, _ = orc.pack(cs, with_cands=True, t_opt_bp=10000)
    assert st == orc.OK
    assert info.scale_index != _m_star(37, 10, 64, 64)
    assert (pl["scale_den"] == 1 << 20).all()


HYBRID = ([chartgen.small_case(s, n=400, family="tss", side=512, rho=0.6) for s in range(2)] +
          [chartgen.small_case(s, n=300, family="lightmap", side=384, rho=0.9) for s in range(2)])


@pytest.mark.parametrize("t", [100, 300, 1000])
@pytest.mark.parametrize("cs", HYBRID, ids=lambda c: c.name)
def test_exact_tail_valid_and_uniform(orc, cs, t):
    st, pl, info, cands = orc.pack(cs, with_cands=True, t_opt_bp=t, flags=orc.F_EXACT_TAIL)
    assert st == orc.OK
    m = info.scale_index
    assert (pl["scale_num"] == m).all() and (pl["scale_den"] == cs.scale_count).all()
    assert info.l2_stretch == cs.scale_count / m
    assert int((pl["mode"] == 1).sum()) == (cs.n_charts - cands[m - 1].switched_at
                                            if cands[m - 1].switched_at >= 0 else 0)
    assert orc.validate(cs, pl) == {"overlap": 0, "gutter": 0, "oob": 0}
    succ = [i + 1 for i, c in enumerate(cands) if c.success]
    assert m == max(succ)  # every chart at m/M: the area-weighted choice is the largest m


def test_exact_tail_not_worse_than_prefix(orc):
    better = 0
    for cs in HYBRID:
        for t in (300, 1000):
            _, _, ie, _ = orc.pack(cs, with_cands=True, t_opt_bp=t, flags=orc.F_EXACT_TAIL)
            _, _, ip, _ = orc.pack(cs, with_cands=True, t_opt_bp=t)
            assert ie.l2_stretch <= ip.l2_stretch + 1e-12, (cs.name, t)
            better += ie.l2_stretch < ip.l2_stretch - 1e-9
    assert better >= 3
