"""Seeded random parity sweep: the CUDA path against the oracle over the spec
space a user can reach -- chart families (UV, TSS, lightmap, mixed), counts
and atlas sizes that span one to many rows and several raster tiles, fill
ratios from trivial fits to heavy downscaling, the quality knob k, gutters,
M, the hybrid threshold t_opt and every flag combination that the method
defines (pre-rotation, exact tail, ablations, paper-literal locks).  Each case
is compared element by element (proxies, order, every evaluated candidate,
placements; stretch within 1e-6) by test_gpu_parity._compare_pack, and every
packing is checked overlap-free by the GPU validator (P:85 / P:1025).

The parameters are drawn from chartgen.SplitMix64 with a fixed seed, so the
sweep is the same on every run; NTABI_FUZZ=<n> widens it locally.
"""
import os

import pytest

import chartgen
from test_gpu_parity import _compare_pack, ctx  # noqa: F401  (the module-scoped context fixture)

pytestmark = pytest.mark.gpu

N = int(os.environ.get("NTABI_FUZZ", "160"))
FAMILIES = ["uv", "tss", "lightmap", "mixed"]
FLAG_SETS = [0, 0, 0, 8, 32, 1, 2, 3, 16, 8 | 2, 4, 32 | 8]


def case(i):
    r = chartgen.SplitMix64(0xF00D + i)
    fam = FAMILIES[r.randint(0, len(FAMILIES) - 1)]
    side = [128, 256, 512, 1024][r.randint(0, 3)]
    n = r.randint(8, 260 if side >= 512 else 140)
    rho = 0.2 + 1.6 * r.uniform()
    cs = chartgen.small_case(i, n=n, side=side, family=fam, rho=rho)
    kw = dict(local_aabb_count=[1, 2, 5, 10, 17][r.randint(0, 4)],
              gutter=[0, 1, 1, 1, 2][r.randint(0, 4)],
              scale_count=[16, 32, 64, 64, 64][r.randint(0, 4)],
              flags=FLAG_SETS[r.randint(0, len(FLAG_SETS) - 1)])
    if r.uniform() < 0.3 or kw["flags"] & 32:
        kw["t_opt_bp"] = [50, 300, 1000, 3000][r.randint(0, 3)]
    if kw["flags"] & 16:   # NO_OBB is an ablation of the plain-AABB modes
        kw["local_aabb_count"] = 1
    return cs, kw


@pytest.mark.parametrize("i", range(N))
def test_random_spec_parity(orc, ctx, i):
    cs, kw = case(i)
    st = _compare_pack(orc, ctx, cs, check_profiles=2, **kw)
    if st == orc.OK:
        from paper_2602_07782_b200 import spec_of
        _, pl, _ = ctx.pack(cs.xy, cs.start, spec_of(cs, **kw))
        g = kw.get("gutter", cs.gutter)
        m = ctx.validate(cs.xy, cs.start, pl, cs.atlas_w, cs.atlas_h, gutter=g)
        if not kw["flags"] & 4:  # (the paper-literal locks admit overlaps, LOCK-1)
            assert m["overlap"] == m["gutter"] == m["oob"] == 0, (cs.name, kw, m)


def large_case(i):
    r = chartgen.SplitMix64(0xB16 + i)
    fam = FAMILIES[r.randint(0, len(FAMILIES) - 1)]
    side = [2048, 4096][r.randint(0, 1)]
    n = r.randint(400, 3000)
    rho = 0.3 + 1.4 * r.uniform()
    cs = chartgen.generate(fam, n, side, side, 7000 + i, rho=rho, side_limit=side / 4,
                           name=f"large-{fam}-n{n}-s{i}")
    kw = dict(local_aabb_count=[2, 5, 10, 10][r.randint(0, 3)],
              flags=[0, 0, 8, 32, 3][r.randint(0, 4)])
    if r.uniform() < 0.4 or kw["flags"] & 32:
        kw["t_opt_bp"] = [100, 500, 2000][r.randint(0, 2)]
    return cs, kw


@pytest.mark.parametrize("i", range(10))
def test_random_large_parity(orc, ctx, i):
    """Larger random sets (400-3,000 charts, 2048^2 / 4096^2): many raster
    tiles per candidate, several position windows per fold, long rows."""
    cs, kw = large_case(i)
    _compare_pack(orc, ctx, cs, check_profiles=1, **kw)


def batch_case(i):
    r = chartgen.SplitMix64(0xBA7C + i)
    side = [256, 512, 1024][r.randint(0, 2)]
    sets = []
    for j in range(r.randint(2, 24)):
        fam = FAMILIES[r.randint(0, len(FAMILIES) - 1)]
        sets.append(chartgen.small_case(100 * i + j, n=r.randint(1, 180), side=side, family=fam,
                                        rho=0.2 + 1.8 * r.uniform()))
    kw = dict(local_aabb_count=[1, 5, 10][r.randint(0, 2)], flags=[0, 0, 8, 3][r.randint(0, 3)])
    if r.uniform() < 0.2:
        kw["t_opt_bp"] = 500  # hybrid atlases go through tabi_pack ("solo")
    return sets, kw


@pytest.mark.parametrize("i", range(12))
def test_random_batch_parity(orc, ctx, i):
    """tabi_pack_many on random batches (1-180 charts per atlas, mixed
    families, fill ratios from trivial to NO_FIT): every atlas's status and
    placements equal the oracle's pack of that atlas alone."""
    import numpy as np
    from paper_2602_07782_b200 import OK, concat_chart_sets, spec_of
    sets, kw = batch_case(i)
    xy, cst, abase, res = concat_chart_sets(sets)
    st, pl, infos, ast, bi = ctx.pack_many(xy, cst, abase, spec_of(sets[0], **kw), res_xy=res,
                                           raise_on_error=False)
    for a, cs in enumerate(sets):
        st_o, pl_o, info_o, _ = orc.pack(cs, **kw)
        assert ast[a] == st_o, (i, a, ast[a], st_o)
        if st_o == OK:
            assert infos[a].scale_index == info_o.scale_index, (i, a)
            assert pl[abase[a]:abase[a + 1]].tobytes() == np.ascontiguousarray(pl_o).tobytes(), (i, a)


def edge_case(i):
    """Hand-shaped extremes mixed at random: slivers (aspect up to 1:200),
    sub-texel and one-texel charts, charts close to the atlas size, stars with
    up to 300 vertices (beyond the proxy kernel's shared-memory vertex cache),
    far-off-origin coordinates, both windings, duplicate consecutive vertices
    and collinear runs (valid simple outlines)."""
    import math
    r = chartgen.SplitMix64(0xED6E + i)
    side = [64, 256, 1024][r.randint(0, 2)]
    polys = []
    for _ in range(r.randint(1, 60)):
        kind = r.randint(0, 6)
        ox, oy = r.uniform(-5000, 5000), r.uniform(-5000, 5000)
        if kind == 0:    # sliver
            L, t = r.uniform(4, side * 0.9), r.uniform(0.05, 2.0)
            p = [(0, 0), (L, 0), (L, t), (0, t)]
        elif kind == 1:  # sub-texel / one-texel
            a = r.uniform(0.02, 1.0)
            p = [(0, 0), (a, 0), (a, a), (0, a)]
        elif kind == 2:  # near the atlas size
            a, b = r.uniform(0.3, 0.95) * side, r.uniform(0.1, 0.9) * side
            p = [(0, 0), (a, 0), (a, b), (0, b)]
        elif kind == 3:  # star with many vertices
            nv = r.randint(60, 300)
            R = r.uniform(3, side * 0.3)
            p = [(R * (0.4 + 0.6 * r.uniform()) * math.cos(2 * math.pi * j / nv),
                  R * (0.4 + 0.6 * r.uniform()) * math.sin(2 * math.pi * j / nv)) for j in range(nv)]
        elif kind == 4:  # triangle, clockwise
            a, b = r.uniform(2, side * 0.4), r.uniform(2, side * 0.4)
            p = [(0, 0), (0, b), (a, 0)]
        elif kind == 5:  # collinear runs and a repeated vertex
            a = r.uniform(4, side * 0.3)
            p = [(0, 0), (a / 3, 0), (2 * a / 3, 0), (a, 0), (a, a), (a, a), (0, a)]
        else:            # rotated rectangle
            a, b, th = r.uniform(2, side * 0.3), r.uniform(2, side * 0.3), r.uniform(0, math.pi)
            c, s = math.cos(th), math.sin(th)
            p = [(x * c - y * s, x * s + y * c) for x, y in [(0, 0), (a, 0), (a, b), (0, b)]]
        polys.append([(x + ox, y + oy) for x, y in p])
    cs = chartgen.from_polygons(polys, side, side, name=f"edge-{i}")
    kw = dict(local_aabb_count=[1, 3, 10, 64][r.randint(0, 3)], gutter=[0, 1, 2][r.randint(0, 2)],
              flags=[0, 0, 8, 3, 32][r.randint(0, 4)])
    if r.uniform() < 0.3 or kw["flags"] & 32:
        kw["t_opt_bp"] = [300, 3000][r.randint(0, 1)]
    return cs, kw


@pytest.mark.parametrize("i", range(40))
def test_random_edge_parity(orc, ctx, i):
    cs, kw = edge_case(i)
    _compare_pack(orc, ctx, cs, check_profiles=2, **kw)


@pytest.mark.parametrize("i", range(24))
def test_random_validator_parity(orc, ctx, i):
    """N3 validator on random packings, valid and corrupted (random shifts,
    mirror flips, pre-rotation indices, scales): overlap / gutter / oob /
    covered counts bit-exact against oracle/validate.c, occupancy exact,
    stretch to 1e-12."""
    import numpy as np
    from paper_2602_07782_b200 import spec_of
    cs, kw = case(1000 + i)
    st, pl, _ = ctx.pack(cs.xy, cs.start, spec_of(cs, **kw), raise_on_error=False)
    if st != orc.OK:
        pytest.skip("no packing")
    rng = np.random.default_rng(i)
    g = kw.get("gutter", cs.gutter)
    for trial in range(3):
        bad = pl.copy()
        if trial:
            k = rng.choice(len(bad), size=max(1, len(bad) // (2 + trial)), replace=False)
            bad["tx"][k] += rng.integers(-9, 10, size=len(k))
            bad["ty"][k] += rng.integers(-9, 10, size=len(k))
            bad["mirror_x"][k] ^= rng.integers(0, 2, size=len(k)).astype(bad["mirror_x"].dtype)
            if trial == 2:
                bad["prerot"][k] = rng.integers(0, 8, size=len(k)).astype(bad["prerot"].dtype)
        mo = orc.metrics(cs, bad, gutter=g)
        mg = ctx.validate(cs.xy, cs.start, bad, cs.atlas_w, cs.atlas_h, gutter=g)
        for key in ("overlap", "gutter", "oob", "covered"):
            assert mg[key] == mo[key], (i, trial, key, mg[key], mo[key])
        assert mg["occupancy"] == mo["occupancy"]
        assert mg["l2_stretch"] == pytest.approx(mo["l2_stretch"], rel=1e-12)
        if trial == 0 and not kw["flags"] & 4:
            assert mg["overlap"] == mg["gutter"] == mg["oob"] == 0


@pytest.mark.parametrize("i", range(16))
def test_random_async_parity(orc, ctx, i):
    """tabi_pack_async + tabi_pack_wait on random specs: the bytes and the
    statistics of the synchronous pack (and so of the oracle)."""
    import torch
    from paper_2602_07782_b200 import spec_of
    cs, kw = case(2000 + i)
    xy, start = torch.from_numpy(cs.xy).cuda(), torch.from_numpy(cs.start).cuda()
    st_s, out_s, info_s = ctx.pack(xy, start, spec_of(cs, **kw), raise_on_error=False)
    torch.cuda.synchronize()
    ref = out_s.cpu().numpy().tobytes()
    out = ctx.pack_async(xy, start, spec_of(cs, **kw))
    st, out2, info = ctx.wait(raise_on_error=False)
    torch.cuda.synchronize()
    assert st == st_s and info.scale_index == info_s.scale_index
    if st == orc.OK:
        assert out.cpu().numpy().tobytes() == ref


def test_two_contexts_async_on_two_streams(orc):
    """Distinct contexts may run concurrently (tabi.h): two asynchronous packs
    in flight at once on two streams of one GPU, each equal to the oracle."""
    import numpy as np
    import torch
    from paper_2602_07782_b200 import Context, spec_of
    cases = [case(3000 + j) for j in range(2)]
    ctxs = [Context(0, max_charts=4096, max_vertices=1 << 16, max_atlas_side=4096) for _ in cases]
    streams = [torch.cuda.Stream() for _ in cases]
    outs = []
    for c, s, (cs, kw) in zip(ctxs, streams, cases):
        xy, start = torch.from_numpy(cs.xy).cuda(), torch.from_numpy(cs.start).cuda()
        torch.cuda.synchronize()
        outs.append((xy, start, c.pack_async(xy, start, spec_of(cs, **kw), stream=s.cuda_stream)))
    for c, (xy, start, out), (cs, kw) in zip(ctxs, outs, cases):
        st, _, info = c.wait(raise_on_error=False)
        st_o, pl_o, info_o, _ = orc.pack(cs, with_cands=True, **kw)
        assert st == st_o
        if st == orc.OK:
            torch.cuda.synchronize()
            assert out.cpu().numpy().tobytes() == np.ascontiguousarray(pl_o).tobytes()
    for c in ctxs:
        c.close()
