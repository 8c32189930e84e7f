"""CUDA path (through the C ABI) vs the CPU oracle, element by element.

Bar (BASELINE.json north_star): proxies, order, footprints, offsets, lock
flags, per-candidate outcomes, row statistics and placements bit-exact;
scale and stretch within 1e-6 relative.  Small cases span several rows,
knees and ragged tails; full-size C3 (1,572 charts, 4096^2) is compared in
full (the oracle finishes it in seconds).
"""
import numpy as np
import pytest

import chartgen

pytestmark = pytest.mark.gpu

PROXY_FIELDS = ("w", "h", "area2", "xmin", "ymin", "rot90", "fx", "fy", "obb_j", "prerot", "umin",
                "umax", "vmin", "vmax")


@pytest.fixture(scope="module")
def ctx():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    from paper_2602_07782_b200 import Context
    c = Context(0, max_charts=25000, max_vertices=1 << 19, max_atlas_side=16384)
    yield c
    c.close()


def _compare_pack(orc, ctx, cs, res=(1.0, 1.0), check_profiles=0, **kw):
    import oracle
    from paper_2602_07782_b200 import spec_of
    st_o, pl_o, info_o, cands_o = oracle.pack(cs, res=res, with_cands=True, **kw)
    st_g, pl_g, info_g = ctx.pack(cs.xy, cs.start, spec_of(cs, **kw), res=res)
    assert st_g == st_o, (st_g, st_o)
    if st_o != oracle.OK:
        return st_o
    n = cs.n_charts
    M = kw.get("scale_count", cs.scale_count)
    k = kw.get("local_aabb_count", cs.local_aabb_count)
    g = kw.get("gutter", cs.gutter)
    # proxies (D3-D8) bit-exact
    st, px, _ = oracle.build_proxies(cs.xy, cs.start, k, res, flags=kw.get("flags", 0))
    gp = ctx.proxies(n)
    for f in PROXY_FIELDS:
        assert np.array_equal(gp[f], np.array([getattr(p, f) for p in px])), f
    for f in ("top", "bot", "left", "right"):
        assert np.array_equal(gp[f][:, :k], np.array([list(getattr(p, f))[:k] for p in px])), f
    # order (D9)
    perm_o = oracle.sort_order(px)
    assert np.array_equal(ctx.perm(n), perm_o)
    # per-candidate outcomes
    gc = ctx.candidates(M)
    # the GPU evaluates candidate waves below the area bound; every
    # evaluated candidate must agree with the exhaustive oracle, and the winner is
    # the oracle's largest successful m
    assert gc["evaluated"].sum() >= 1
    assert info_g.scale_index == info_o.scale_index
    for m in range(1, M + 1):
        co = cands_o[m - 1]
        if not gc["evaluated"][m - 1]:
            assert m < info_g.scale_index or not co.success, m
            continue
        assert gc["success"][m - 1] == co.success, m
        if co.success:
            for f in ("score", "rows", "knees_found", "knee_rows", "prefix_rows", "p",
                      "switched_at"):
                assert gc[f][m - 1] == getattr(co, f), (m, f)
    # placements bit-exact, scale/stretch
    for f in ("tx", "ty", "scale_num", "scale_den", "box_w", "box_h", "rot90", "flip_x", "flip_y",
              "mirror_x", "mode", "prerot"):
        assert np.array_equal(pl_g[f], pl_o[f]), f
    assert info_g.scale_index == info_o.scale_index
    assert info_g.l2_stretch == pytest.approx(info_o.l2_stretch, rel=1e-6)
    assert (info_g.rows, info_g.knees_found, info_g.knee_rows) == (
        info_o.rows, info_o.knees_found, info_o.knee_rows)
    # footprints and offsets on sampled candidates / charts
    if check_profiles:
        rng = chartgen.SplitMix64(n * 7 + M)
        ms = sorted({M, info_o.scale_index, max(1, M // 3), rng.randint(1, M)})
        for m in ms:
            if not gc["evaluated"][m - 1] or (not gc["success"][m - 1]
                                                 and not cands_o[m - 1].success):
                continue
            off_g, lk_g = ctx.offsets(m, n)
            ss = sorted({0, n - 1, *[rng.randint(0, n - 1) for _ in range(check_profiles)]})
            r0 = int(gc["switched_at"][m - 1])
            r0 = n if r0 < 0 else r0

            def scale(pos):  # tail charts were re-rasterized at p / 2^20 (D24)
                return (int(gc["p"][m - 1]), 1 << 20) if pos >= r0 else (m, M)

            for s in ss:
                prof = ctx.profile(m, s)
                po = oracle.Profile(px[perm_o[s]], *scale(s), g)
                assert prof is not None
                Wd, Hd, dt, db, dl, dr = prof
                assert (Wd, Hd) == (po.Wd, po.Hd)
                assert np.array_equal(dt, po.Dtop) and np.array_equal(db, po.Dbot)
                assert np.array_equal(dl, po.Dleft) and np.array_equal(dr, po.Dright)
                if s + 1 < n:
                    pn = oracle.Profile(px[perm_o[s + 1]], *scale(s), g)
                    if s < r0:
                        po = oracle.Profile(px[perm_o[s]], m, M, g)
                    off = oracle.offset(po, pn)
                    assert off_g[s] == off
                    la, lb = oracle.locks(po, pn, off) if off < po.Wd else (False, False)
                    assert lk_g[s] == (1 if la else 0) | (2 if lb else 0)
    return st_o


SMALL = ([chartgen.config1a(s) for s in range(6)] + [chartgen.config1b(s) for s in range(6)] +
         [chartgen.small_case(s, n=48) for s in range(4)] +
         [chartgen.small_case(s, n=48, family="uv") for s in range(4)] +
         [chartgen.small_case(s, n=64, family="mixed", rho=1.2) for s in range(3)] +
         [chartgen.small_case(s, n=200, family="uv", side=512, rho=0.9) for s in range(2)])


@pytest.mark.parametrize("cs", SMALL, ids=lambda c: c.name)
def test_small_parity(orc, ctx, cs):
    _compare_pack(orc, ctx, cs, check_profiles=6)


@pytest.mark.parametrize("seed", range(3))
def test_config2_parity(orc, ctx, seed):
    _compare_pack(orc, ctx, chartgen.config2(seed), check_profiles=8)


@pytest.mark.parametrize("rho", [0.5, 2.0])
def test_config3_full_size_parity(orc, ctx, rho):
    cs = chartgen.config3(0, rho=rho)
    _compare_pack(orc, ctx, cs, check_profiles=16)
    import oracle
    from paper_2602_07782_b200 import spec_of
    _, pl, _ = ctx.pack(cs.xy, cs.start, spec_of(cs))
    assert oracle.validate(cs, pl) == {"overlap": 0, "gutter": 0, "oob": 0}


@pytest.mark.parametrize("k", [1, 2, 5, 17, 64])
def test_quality_knob_parity(orc, ctx, k):
    _compare_pack(orc, ctx, chartgen.small_case(11, n=60, family="uv"), check_profiles=4,
                  local_aabb_count=k)


@pytest.mark.parametrize("kw", [dict(gutter=0), dict(gutter=3), dict(scale_count=1),
                                dict(scale_count=17), dict(scale_count=256),
                                dict(flags=1), dict(flags=2), dict(flags=4), dict(flags=16),
                                dict(flags=16, local_aabb_count=1)],
                         ids=lambda d: "-".join(f"{a}{b}" for a, b in d.items()))
def test_spec_variants_parity(orc, ctx, kw):
    _compare_pack(orc, ctx, chartgen.small_case(5, n=50, family="mixed", rho=0.8),
                  check_profiles=3, **kw)


PREROT = ([chartgen.small_case(s, n=48, family="uv") for s in range(3)] +
          [chartgen.small_case(s, n=300, family="tss", side=512, rho=0.6) for s in range(2)] +
          [chartgen.config2(0), chartgen.config3(0)])


@pytest.mark.parametrize("cs", PREROT, ids=lambda c: c.name)
def test_prerotate_parity(orc, ctx, cs):
    """R4 pre-rotation (TABI_F_PREROTATE): angle, rotated proxies, order,
    candidates and placements (prerot included) bit-exact; the packing is valid
    under the validator, which applies step 0 to the original outlines."""
    import oracle
    from paper_2602_07782_b200 import F_PREROTATE, spec_of
    _compare_pack(orc, ctx, cs, check_profiles=4, flags=F_PREROTATE)
    _, pl, _ = ctx.pack(cs.xy, cs.start, spec_of(cs, flags=F_PREROTATE))
    assert (pl["prerot"] > 0).any()
    assert oracle.validate(cs, pl) == {"overlap": 0, "gutter": 0, "oob": 0}


@pytest.mark.parametrize("mode", ["tight_only", "balanced_only", "chameleon"])
@pytest.mark.parametrize("cs", [chartgen.config2(1),
                                chartgen.small_case(0, n=300, family="tss", side=512, rho=0.6)],
                         ids=lambda c: c.name)
def test_ablation_modes_parity(orc, ctx, cs, mode):
    """the paper's ablation / baseline modes run on the
    same kernels, bit-exact against the oracle."""
    from paper_2602_07782_b200 import ABLATIONS
    _compare_pack(orc, ctx, cs, check_profiles=4, **ABLATIONS[mode])


def test_unsnapped_input_with_resolution(orc, ctx):
    """UV input in [0, 1] times a texture resolution: exercises D2 round-half-even."""
    cs = chartgen.small_case(2, n=40, family="uv", side=256)
    rng = np.random.default_rng(0)
    xy = (cs.xy / 256.0 + rng.uniform(-1e-4, 1e-4, cs.xy.shape)).astype(np.float32)
    cs2 = chartgen.ChartSet("uv01", xy, cs.start, 256, 256)
    _compare_pack(orc, ctx, cs2, res=(256.0, 256.0), check_profiles=3)


HYBRID = [chartgen.small_case(s, n=400, family="tss", side=512, rho=0.6) for s in range(2)] + \
         [chartgen.small_case(s, n=300, family="lightmap", side=384, rho=0.9) for s in range(2)] + \
         [chartgen.generate("lightmap", 2500, 2048, 2048, 7, rho=0.8, name="lightmap-2500")]


@pytest.mark.parametrize("t", [100, 300, 1000])
@pytest.mark.parametrize("cs", HYBRID, ids=lambda c: c.name)
def test_hybrid_tail_parity(orc, ctx, cs, t):
    """D23-D26 prefix tail: rows, sigma, placements and the area-weighted
    candidate choice bit-exact; stretch within 1e-6."""
    _compare_pack(orc, ctx, cs, check_profiles=2, t_opt_bp=t)


def test_config4_policy_full_size(orc, ctx):
    """C4: 20,000 lightmap charts into 8192^2 with the paper's t_opt policy
    (1 % for > 10,000 charts): full oracle comparison."""
    _compare_pack(orc, ctx, chartgen.config4(0), check_profiles=0)


def test_config4_sequential_full_size(orc, ctx):
    """C4 as bench.py's --workload C4 times it: 20,000 lightmap charts into
    8192^2 with t_opt = 0 (sequential rows only): full oracle comparison
    (proxies, order, every evaluated candidate, placements)."""
    _compare_pack(orc, ctx, chartgen.config4(0, t_opt_bp=0), check_profiles=0)


@pytest.mark.parametrize("i", [0, 311])
def test_config5_atlas_single_pack(orc, ctx, i):
    """One atlas of the C5 batch workload (200-2,000 tss charts, 2048^2) by
    tabi_pack against the oracle (the batch path is compared in
    test_gpu_many.py)."""
    _compare_pack(orc, ctx, chartgen.config5(i), check_profiles=2)


@pytest.mark.parametrize("t", [100, 1000, 10000])
@pytest.mark.parametrize("cs", HYBRID, ids=lambda c: c.name)
def test_exact_tail_parity(orc, ctx, cs, t):
    """R6 exact-greedy tail: rows, placements (tail charts at
    m/M, mode 1) and the candidate choice bit-exact against the oracle."""
    from paper_2602_07782_b200 import F_EXACT_TAIL
    _compare_pack(orc, ctx, cs, check_profiles=2, t_opt_bp=t, flags=F_EXACT_TAIL)


@pytest.mark.parametrize("kw", [dict(flags=8 | 1), dict(flags=8 | 32, t_opt_bp=300),
                                dict(flags=2 | 4), dict(flags=16 | 2, local_aabb_count=1),
                                dict(flags=32 | 4, t_opt_bp=1000, gutter=0),
                                dict(flags=8 | 16, scale_count=17, gutter=2)],
                         ids=lambda d: "-".join(f"{a}{b}" for a, b in d.items()))
def test_flag_combinations_parity(orc, ctx, kw):
    """Flags together (pre-rotation, exact tail, ablations, paper-literal
    locks) with other spec knobs: bit-exact against the oracle."""
    _compare_pack(orc, ctx, chartgen.small_case(2, n=300, family="tss", side=512, rho=0.6),
                  check_profiles=2, **kw)


def test_exact_tail_config4_full_size(orc, ctx):
    from paper_2602_07782_b200 import F_EXACT_TAIL, spec_of
    cs = chartgen.config4(0)
    _compare_pack(orc, ctx, cs, check_profiles=0, flags=F_EXACT_TAIL)
    _, pl, info = ctx.pack(cs.xy, cs.start, spec_of(cs, flags=F_EXACT_TAIL))
    assert info.prefix_rows > 0 and (pl["mode"] == 1).any()
    m = ctx.validate(cs.xy, cs.start, pl, cs.atlas_w, cs.atlas_h, gutter=cs.gutter)
    assert m["overlap"] == m["gutter"] == m["oob"] == 0


@pytest.mark.parametrize("wave", ["1", "3", "256"])
def test_wave_sizes(orc, ctx, wave, monkeypatch):
    """Candidate waves of any size give the exhaustive result: 1 = one candidate
    per wave (many host round trips), 256 = all candidates at once."""
    monkeypatch.setenv("TABI_WAVE", wave)
    for cs in (chartgen.config1b(2), chartgen.small_case(4, n=60, family="mixed", rho=1.3)):
        _compare_pack(orc, ctx, cs, check_profiles=3)


@pytest.mark.parametrize("fused", ["0", "1"])
def test_fused_and_split_paths(orc, ctx, fused, monkeypatch):
    """The fused persistent wave kernel (default) and the split K3 / K3b / K4
    launches (TABI_FUSED=0) both agree with the oracle, hybrid tail included."""
    monkeypatch.setenv("TABI_FUSED", fused)
    cases = (chartgen.config2(1), chartgen.small_case(7, n=200, family="uv", side=512, rho=0.9))
    for cs in cases:
        _compare_pack(orc, ctx, cs, check_profiles=6)
    _compare_pack(orc, ctx, HYBRID[2], check_profiles=2, t_opt_bp=300)
    from paper_2602_07782_b200 import spec_of
    _, _, info = ctx.pack(cases[0].xy, cases[0].start, spec_of(cases[0]))
    assert info.fused == int(fused)


def test_large_chart_path(orc, ctx):
    """Charts whose footprint exceeds the K3 tile buffer (> 8192 cells) take the
    warp-per-chart path; both must agree with the oracle."""
    big = [[(0, 0), (300, 40), (260, 9000), (10, 8800)],
           [(0, 0), (7000, 0), (7000, 2500), (3000, 2600), (0, 2500)]]
    small = [chartgen.config1a(3).polygon(c).tolist() for c in range(10)]
    cs = chartgen.from_polygons(big + small, 16384, 16384)
    _compare_pack(orc, ctx, cs, check_profiles=4, scale_count=8)


def test_long_row_window(orc, ctx):
    """Rows longer than the fold's position window (1,024 sorted positions):
    3,000 small charts fit one 16,384-wide row, so the fold slides its window
    on within the row (same prefix frame); also ragged chart sizes."""
    rng = np.random.default_rng(3)
    polys = []
    for _ in range(3000):
        a, b = int(rng.integers(1, 4)), int(rng.integers(1, 4))
        polys.append([(0, 0), (a, 0), (a, b), (0, b)])
    cs = chartgen.from_polygons(polys, 16384, 64)
    _compare_pack(orc, ctx, cs, check_profiles=0)
    _compare_pack(orc, ctx, cs, check_profiles=0, scale_count=8)


def test_lock1_both_modes(orc, ctx):
    A = [(0, 0), (20, 0), (20, 150), (0, 150)]
    c0 = [(0, 0), (10, 0), (10, 45), (40, 45), (40, 47), (10, 47), (10, 100), (0, 100)]
    c1 = [(0, 0), (10, 0), (10, 35), (0, 35)]
    c2 = [(0, 0), (10, 0), (10, 30), (0, 30)]
    cs = chartgen.from_polygons([A, c0, c1, c2], 40, 256, gutter=0)
    _compare_pack(orc, ctx, cs, flags=4)
    _compare_pack(orc, ctx, cs, flags=0)


def test_single_and_no_fit(orc, ctx):
    from paper_2602_07782_b200 import NO_FIT, spec_of
    cs = chartgen.from_polygons([[(0, 0), (100, 0), (100, 100), (0, 100)]], 64, 64)
    _compare_pack(orc, ctx, cs)
    cs = chartgen.from_polygons([[(0, 0), (10000, 0), (10000, 1), (0, 1)]], 64, 64)
    st, _, info = ctx.pack(cs.xy, cs.start, spec_of(cs))
    assert st == NO_FIT and info.scale_index == 0


def test_invalid_chart_reported(ctx):
    from paper_2602_07782_b200 import EINVAL, spec_of
    cs = chartgen.from_polygons([[(0, 0), (1, 0), (1, 1)], [(0, 0), (5, 0), (10, 0)],
                                 [(0, 0), (2, 0), (2, 2)]], 64, 64)
    st, _, info = ctx.pack(cs.xy, cs.start, spec_of(cs), raise_on_error=False)
    assert st == EINVAL and info.bad_chart == 1
    cs = chartgen.from_polygons([[(0, 0), (1, 0), (1, 1)], [(0, 0), (5, 0), (10, 3)],
                                 [(0, 0), (2, 0), (2, 2)]], 64, 64)
    bad = cs.xy.copy()
    bad[13] = np.nan  # y of chart 2's first vertex
    st, _, info = ctx.pack(bad, cs.start, spec_of(cs), raise_on_error=False)
    assert st == EINVAL and info.bad_chart == 2


def test_device_inputs_match_host(ctx):
    import torch
    from paper_2602_07782_b200 import PLACEMENT_DTYPE, spec_of
    cs = chartgen.config2(1)
    st_h, pl_h, info_h = ctx.pack(cs.xy, cs.start, spec_of(cs))
    xy = torch.from_numpy(cs.xy).cuda()
    start = torch.from_numpy(cs.start).cuda()
    st_d, out_d, info_d = ctx.pack(xy, start, spec_of(cs))
    torch.cuda.synchronize()
    pl_d = out_d.cpu().numpy().view(PLACEMENT_DTYPE)
    assert st_h == st_d and info_h.scale_index == info_d.scale_index
    assert pl_h.tobytes() == pl_d.tobytes()


def test_pack_batch_equals_single_packs(ctx):
    """tabi_pack_batch (two contexts / host threads on one GPU here) gives the
    same bytes as packing each atlas alone (S:457 determinism across jobs)."""
    from paper_2602_07782_b200 import Context, OK, pack_batch, spec_of
    sets = [chartgen.config5(i) for i in range(6)]
    c2 = Context(0, max_charts=2100, max_vertices=1 << 17, max_atlas_side=2048)
    c3 = Context(0, max_charts=2100, max_vertices=1 << 17, max_atlas_side=2048)
    st, outs, infos = pack_batch([c2, c3], sets, [spec_of(cs) for cs in sets])
    assert st == OK
    for cs, pl, inf in zip(sets, outs, infos):
        st1, pl1, inf1 = ctx.pack(cs.xy, cs.start, spec_of(cs))
        assert st1 == OK and inf.scale_index == inf1.scale_index
        assert pl.tobytes() == pl1.tobytes()
    c2.close()
    c3.close()


@pytest.mark.parametrize("path", ["default", "bitonic", "chunk", "rank", "radix"])
def test_sort_paths_with_ties(orc, ctx, path, monkeypatch):
    """D9 order (h desc, w desc, index asc) through each sort path (default:
    the register bitonic network for N <= 2048, the chunked bitonic + merge
    ranks above; TABI_SORT forces the smem bitonic (N <= 4096), chunked, rank or
    radix path), on inputs full of exact (h, w) ties: index order must decide
    them.  N = 900 (one chunk) and 5000 (three chunks, ties across chunks)."""
    import oracle
    from paper_2602_07782_b200 import spec_of
    if path == "default":
        monkeypatch.delenv("TABI_SORT", raising=False)
    else:
        monkeypatch.setenv("TABI_SORT", path)
    rng = np.random.default_rng(5)
    for n in (900, 5000):
        polys = []
        for i in range(n):
            w, h = [(8, 8), (8, 12), (12, 8), (5, 20)][rng.integers(0, 4)]
            if rng.random() < 0.2:
                w, h = int(rng.integers(3, 30)), int(rng.integers(3, 30))
            polys.append([(0, 0), (w, 0), (w, h), (0, h)])
        cs = chartgen.from_polygons(polys, 2048, 2048)
        ctx.pack(cs.xy, cs.start, spec_of(cs, scale_count=4))
        _, px, _ = oracle.build_proxies(cs.xy, cs.start, cs.local_aabb_count, (1.0, 1.0))
        assert np.array_equal(ctx.perm(cs.n_charts), oracle.sort_order(px)), n
    _compare_pack(orc, ctx, chartgen.config2(2), check_profiles=0)


@pytest.mark.parametrize("lanes", ["8", "16", "32"])
def test_proxy_lane_groups(orc, ctx, lanes, monkeypatch):
    """K1 with 8, 16 and 32 lanes per chart (TABI_PROXY_LANES forces the
    group size the launcher otherwise picks by chart count): proxies, order
    and the whole pack bit-exact, on charts from 3 to ~100 vertices."""
    monkeypatch.setenv("TABI_PROXY_LANES", lanes)
    _compare_pack(orc, ctx, chartgen.small_case(9, n=120, family="mixed", rho=0.9),
                  check_profiles=2)
    _compare_pack(orc, ctx, chartgen.small_case(4, n=60, family="uv"), check_profiles=2,
                  local_aabb_count=64)


def test_determinism_and_capacity_growth():
    from paper_2602_07782_b200 import Context, spec_of
    cs = chartgen.config3(1, rho=2.0)
    small = Context(0, max_charts=cs.n_charts, max_vertices=cs.n_vertices, max_atlas_side=4096)
    outs = [small.pack(cs.xy, cs.start, spec_of(cs))[1].tobytes() for _ in range(3)]
    assert outs[0] == outs[1] == outs[2]
    small.close()


@pytest.mark.parametrize("a,n,W,g,M", [(30, 400, 1024, 1, 64), (30, 10, 1024, 1, 64),
                                       (17, 700, 512, 2, 32), (9, 900, 256, 1, 16)])
def test_prefix_tail_equal_squares_parity(orc, ctx, a, n, W, g, M):
    """The closed-form tail family of tests/test_oracle_tail_closed_form.py
    (every chart in the D24 tail; sigma rule, its cap, re-layout rounds, the
    D25 choice) through the GPU: graph rounds loop, tail kernels, prefix rows."""
    polys = [[(0, 0), (a, 0), (a, a), (0, a)] for _ in range(n)]
    cs = chartgen.from_polygons(polys, W, W)
    _compare_pack(orc, ctx, cs, check_profiles=3, t_opt_bp=1000, gutter=g, scale_count=M)


def test_obb_angle_ties_parity(orc, ctx):
    """D6's tie rule on the GPU: shapes whose two best OBB angles tie exactly
    (tests/test_oracle_properties.py::D6_TIES), packed together with a few
    scaled copies -- proxies (obb_j, extents) and placements bit-exact."""
    from test_oracle_properties import D6_TIES
    polys = []
    for s in (1, 2, 3):
        polys += [[(x * s, y * s) for x, y in p] for p in D6_TIES]
    cs = chartgen.from_polygons(polys, 1024, 1024)
    _compare_pack(orc, ctx, cs, check_profiles=4)


@pytest.mark.parametrize("sort_path", ["default", "rank"])
def test_multi_cta_slot_layout(ctx, monkeypatch, sort_path):
    """The slot layout for 4096 < N <= 2^17 runs as one CTA per 4096 sorted
    positions with decoupled look-back (prep_multi_kernel): the same packs
    and winning candidate record as the one-CTA prep_kernel
    (TABI_PREP_MULTI=0), at ragged sizes (one position past a block, several
    blocks, C4's 20,000), from the chunked sort's keys and from the rank sort
    (no sorted keys: perm loads), twice in a row (the look-back epochs)."""
    from paper_2602_07782_b200 import spec_of
    if sort_path != "default":
        monkeypatch.setenv("TABI_SORT", sort_path)
    for cs in (chartgen.generate("lightmap", 4097, 4096, 4096, 3, rho=0.8),
               chartgen.generate("tss", 9000, 8192, 8192, 4, rho=1.2),
               chartgen.config4(0, t_opt_bp=0)):
        sp = spec_of(cs)
        monkeypatch.setenv("TABI_PREP_MULTI", "0")
        st0, pl0, info0 = ctx.pack(cs.xy, cs.start, sp)
        c0 = ctx.candidates(cs.scale_count)
        monkeypatch.delenv("TABI_PREP_MULTI")
        for _ in range(2):
            st1, pl1, info1 = ctx.pack(cs.xy, cs.start, sp)
            c1 = ctx.candidates(cs.scale_count)
            assert st0 == st1 and info0.scale_index == info1.scale_index, cs.name
            assert pl0.tobytes() == pl1.tobytes(), cs.name
            w = info0.scale_index - 1  # (the winner's record: aborted lower
            assert c0[w].tobytes() == c1[w].tobytes(), cs.name  # candidates are schedule-dependent)


def test_proxy_fork_is_exact(orc, ctx, monkeypatch):
    """The prologue fork (sizes_kernel -> order -> slot layout on the pack's
    stream while proxy_kernel runs on a second one; default above 4,096
    charts): forced on for small packs it matches the oracle, and a bad chart
    (zero area: collinear outlines) is reported with the same index as without
    the fork."""
    from paper_2602_07782_b200 import spec_of
    monkeypatch.setenv("TABI_PROXY_FORK", "1")
    _compare_pack(orc, ctx, chartgen.config2(1), check_profiles=0)
    _compare_pack(orc, ctx, chartgen.config3(1, rho=2.0), check_profiles=0)
    sq = [(0, 0), (10, 0), (10, 10), (0, 10)]
    for bad in ([(0, 0), (5, 0), (9, 0)], [(0, 0), (5, 5), (10, 10), (3, 3)]):
        cs = chartgen.from_polygons([sq, sq, bad, sq, bad], 512, 512)
        res = []
        for f in ("1", "0"):
            monkeypatch.setenv("TABI_PROXY_FORK", f)
            st, _, info = ctx.pack(cs.xy, cs.start, spec_of(cs), raise_on_error=False)
            res.append((st, info.bad_chart))
        assert res[0] == res[1] and res[0][1] == 2, res
