"""GPU validator + metrics (tabi_validate) against the oracle
validator: every count bit-exact, occupancy exact, stretch to 1e-12.

Cases: valid packings (all counts zero, covered > 0) from both paths, and
corrupted placements (shifted, mirrored, pre-rotated, hanging over the edge,
random) so that overlap / gutter / oob are non-zero; gutters 0, 1, 3;
hybrid-tail placements (scale p / 2^20); device-pointer inputs; errors.
"""
import numpy as np
import pytest

import chartgen

pytestmark = pytest.mark.gpu

KEYS = ("overlap", "gutter", "oob", "covered")


@pytest.fixture(scope="module")
def ctx():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    from paper_2602_07782_b200 import Context
    c = Context(0, max_charts=25000, max_vertices=1 << 19, max_atlas_side=16384)
    yield c
    c.close()


def _check(orc, ctx, cs, pl, res=(1.0, 1.0), gutter=None):
    g = cs.gutter if gutter is None else gutter
    mo = orc.metrics(cs, pl, res=res, gutter=g)
    mg = ctx.validate(cs.xy, cs.start, pl, cs.atlas_w, cs.atlas_h, gutter=g, res=res)
    for k in KEYS:
        assert mg[k] == mo[k], (k, mg[k], mo[k])
    assert mg["occupancy"] == mo["occupancy"]
    assert mg["l2_stretch"] == pytest.approx(mo["l2_stretch"], rel=1e-12)
    assert mg["gpu_launches"] >= 3
    return mg


def _corrupt(pl, seed, W, H):
    rng = np.random.default_rng(seed)
    bad = pl.copy()
    n = len(bad)
    idx = rng.choice(n, size=max(1, n // 3), replace=False)
    bad["tx"][idx] += rng.integers(-6, 7, size=len(idx))
    bad["ty"][idx] += rng.integers(-6, 7, size=len(idx))
    bad["mirror_x"][idx] ^= 1
    bad["tx"][0] = W - 2  # hangs over the right edge
    bad["ty"][-1] = -1
    return bad


CASES = ([chartgen.small_case(s, n=48, family="uv") for s in range(3)] +
         [chartgen.small_case(s, n=64, family="mixed", rho=1.2) for s in range(2)] +
         [chartgen.config2(0)])


@pytest.mark.parametrize("cs", CASES, ids=lambda c: c.name)
def test_valid_and_corrupted(orc, ctx, cs):
    from paper_2602_07782_b200 import spec_of
    _, pl, info = ctx.pack(cs.xy, cs.start, spec_of(cs))
    m = _check(orc, ctx, cs, pl)
    assert m["overlap"] == m["gutter"] == m["oob"] == 0 and m["covered"] > 0
    assert m["l2_stretch"] == pytest.approx(info.l2_stretch, rel=1e-12)
    for seed in range(2):
        bad = _corrupt(pl, seed, cs.atlas_w, cs.atlas_h)
        for g in (0, 1, 3):
            m = _check(orc, ctx, cs, bad, gutter=g)
            assert m["overlap"] + m["oob"] > 0


def test_prerotated_and_hybrid(orc, ctx):
    from paper_2602_07782_b200 import F_PREROTATE, spec_of
    cs = chartgen.small_case(1, n=300, family="tss", side=512, rho=0.6)
    _, pl, _ = ctx.pack(cs.xy, cs.start, spec_of(cs, flags=F_PREROTATE))
    assert (pl["prerot"] > 0).any()
    _check(orc, ctx, cs, pl)
    _check(orc, ctx, cs, _corrupt(pl, 5, cs.atlas_w, cs.atlas_h))
    _, pl, info = ctx.pack(cs.xy, cs.start, spec_of(cs, t_opt_bp=300))
    assert info.prefix_rows > 0 and (pl["mode"] == 1).any()
    m = _check(orc, ctx, cs, pl)
    assert m["overlap"] == m["gutter"] == m["oob"] == 0
    assert m["l2_stretch"] == pytest.approx(info.l2_stretch, rel=1e-9)


def test_random_placements(orc, ctx):
    cs = chartgen.small_case(4, n=80, family="uv")
    rng = np.random.default_rng(9)
    from paper_2602_07782_b200 import PLACEMENT_DTYPE
    pl = np.zeros(cs.n_charts, dtype=PLACEMENT_DTYPE)
    pl["tx"] = rng.integers(-20, cs.atlas_w, cs.n_charts)
    pl["ty"] = rng.integers(-20, cs.atlas_h, cs.n_charts)
    pl["scale_num"] = rng.integers(1, 65, cs.n_charts)
    pl["scale_den"] = 64
    pl["box_w"] = rng.integers(1, 40, cs.n_charts)
    pl["rot90"] = rng.integers(0, 2, cs.n_charts)
    pl["flip_x"] = rng.integers(0, 2, cs.n_charts)
    pl["flip_y"] = rng.integers(0, 2, cs.n_charts)
    pl["mirror_x"] = rng.integers(0, 2, cs.n_charts)
    pl["prerot"] = rng.integers(0, 8, cs.n_charts)
    m = _check(orc, ctx, cs, pl)
    assert m["overlap"] > 0 and m["oob"] > 0


def test_full_size_c3_c4(orc, ctx):
    from paper_2602_07782_b200 import spec_of
    for cs in (chartgen.config3(0), chartgen.config4(0)):
        _, pl, info = ctx.pack(cs.xy, cs.start, spec_of(cs))
        m = ctx.validate(cs.xy, cs.start, pl, cs.atlas_w, cs.atlas_h, gutter=cs.gutter)
        assert m["overlap"] == m["gutter"] == m["oob"] == 0
        assert m["l2_stretch"] == pytest.approx(info.l2_stretch, rel=1e-9)
        assert 0.2 < m["occupancy"] < 1.0
    # C3 against the oracle validator, all counts
    cs = chartgen.config3(0)
    _, pl, _ = ctx.pack(cs.xy, cs.start, spec_of(cs))
    _check(orc, ctx, cs, _corrupt(pl, 1, cs.atlas_w, cs.atlas_h))


def test_device_inputs(orc, ctx):
    import torch
    from paper_2602_07782_b200 import spec_of
    cs = chartgen.config2(1)
    _, pl, _ = ctx.pack(cs.xy, cs.start, spec_of(cs))
    bad = _corrupt(pl, 3, cs.atlas_w, cs.atlas_h)
    mh = ctx.validate(cs.xy, cs.start, bad, cs.atlas_w, cs.atlas_h)
    xy = torch.from_numpy(cs.xy).cuda()
    st = torch.from_numpy(cs.start).cuda()
    pd = torch.from_numpy(bad.view(np.uint8).copy()).cuda()
    md = ctx.validate(xy, st, pd, cs.atlas_w, cs.atlas_h)
    for k in KEYS + ("occupancy", "l2_stretch"):
        assert md[k] == mh[k], k


def test_errors(ctx):
    from paper_2602_07782_b200 import EINVAL
    cs = chartgen.small_case(0, n=10, family="uv")
    from paper_2602_07782_b200 import spec_of
    _, pl, _ = ctx.pack(cs.xy, cs.start, spec_of(cs))
    bad = pl.copy()
    bad["scale_num"][4] = 0
    m = ctx.validate(cs.xy, cs.start, bad, cs.atlas_w, cs.atlas_h, raise_on_error=False)
    assert m["status"] == EINVAL and m["bad_chart"] == 4
    m = ctx.validate(cs.xy, cs.start, pl, 0, cs.atlas_h, raise_on_error=False)
    assert m["status"] == EINVAL
    m = ctx.validate(cs.xy, cs.start, pl, cs.atlas_w, cs.atlas_h, gutter=65, raise_on_error=False)
    assert m["status"] == EINVAL


def test_maximum_sizes_self_consistent(ctx):
    """The largest configuration the context allows (25,000 charts, M = 256
    candidate scales, k = 64, a 16,384^2 atlas): too large for the CPU oracle
    in a test, so the GPU result is checked against the GPU validator (no
    overlap, gutter or out-of-bounds texel) and the stretch closed form M/m."""
    from paper_2602_07782_b200 import spec_of
    cs = chartgen.generate("lightmap", 25000, 16384, 16384, 11, rho=0.8, name="max")
    spec = spec_of(cs, scale_count=256, local_aabb_count=64)
    st, pl, info = ctx.pack(cs.xy, cs.start, spec)
    assert st == 0 and info.scale_index >= 1
    assert info.l2_stretch == pytest.approx(256 / info.scale_index, rel=1e-12)
    m = ctx.validate(cs.xy, cs.start, pl, cs.atlas_w, cs.atlas_h, gutter=cs.gutter)
    assert m["overlap"] == m["gutter"] == m["oob"] == 0
    assert m["l2_stretch"] == pytest.approx(info.l2_stretch, rel=1e-9)
