"""Batch mode (tabi_pack_many): many atlases on one GPU
as one device pipeline -- batched proxies, one sort CTA per atlas, and a
persistent kernel whose CTAs take (atlas, candidate) items from a device work
queue.  Every atlas's result must be bit-identical to the CPU oracle's (and to
a single tabi_pack of that atlas), whatever the queue's interleaving."""
import numpy as np
import pytest

import chartgen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    from paper_2602_07782_b200 import Context
    c = Context(0, max_charts=25000, max_vertices=1 << 19, max_atlas_side=8192)
    yield c
    c.close()


def _split(pl, abase):
    return [pl[abase[a]:abase[a + 1]] for a in range(len(abase) - 1)]


def _mixed_sets():
    """Small atlases of several families and fill ratios: some fit at m = 64,
    some need several candidates below the area bound (queue pushes), one has
    a single chart, one is crowded enough to take ~10 candidates."""
    sets = [chartgen.small_case(s, n=40 + 13 * s, family=f, rho=r)
            for s, (f, r) in enumerate([("tss", 0.6), ("uv", 0.9), ("mixed", 1.2), ("tss", 1.6),
                                         ("uv", 0.3), ("tss", 2.4)])]
    sets.append(chartgen.from_polygons([[(0, 0), (30, 0), (30, 12), (0, 12)]], 256, 256))
    sets.append(chartgen.config2(3))
    return sets


def test_pack_many_matches_oracle(orc, ctx):
    import oracle
    from paper_2602_07782_b200 import OK, concat_chart_sets, spec_of
    sets = _mixed_sets()
    # one spec for the batch: the atlas sizes differ, so pack each size group
    for side in sorted({cs.atlas_w for cs in sets}):
        grp = [cs for cs in sets if cs.atlas_w == side]
        xy, cst, abase, res = concat_chart_sets(grp)
        st, pl, infos, ast, bi = ctx.pack_many(xy, cst, abase, spec_of(grp[0]), res_xy=res)
        assert bi.batched_atlases == len(grp) and bi.solo_atlases == 0
        assert bi.candidates_evaluated >= len(grp)
        for cs, part, inf, s in zip(grp, _split(pl, abase), infos, ast):
            st_o, pl_o, info_o, _ = oracle.pack(cs)
            assert s == st_o, (cs.name, s, st_o)
            if st_o != OK:
                continue
            assert inf.scale_index == info_o.scale_index, cs.name
            assert (inf.rows, inf.knees_found, inf.knee_rows) == (
                info_o.rows, info_o.knees_found, info_o.knee_rows), cs.name
            assert abs(inf.l2_stretch - info_o.l2_stretch) <= 1e-6 * info_o.l2_stretch
            assert part.tobytes() == np.ascontiguousarray(pl_o).tobytes(), cs.name


def test_pack_many_c5_equals_single_packs_and_oracle(orc, ctx):
    """24 atlases of the C5 workload (200-2,000 charts, 2048^2): every atlas
    equals its single pack byte for byte; three are also checked against the
    oracle directly."""
    import oracle
    from paper_2602_07782_b200 import OK, concat_chart_sets, spec_of
    sets = [chartgen.config5(i) for i in range(24)]
    xy, cst, abase, res = concat_chart_sets(sets)
    st, pl, infos, ast, bi = ctx.pack_many(xy, cst, abase, spec_of(sets[0]), res_xy=res)
    assert st == OK and bi.batched_atlases == 24
    parts = _split(pl, abase)
    for i, cs in enumerate(sets):
        st1, pl1, inf1 = ctx.pack(cs.xy, cs.start, spec_of(cs))
        assert ast[i] == st1
        assert infos[i].scale_index == inf1.scale_index, i
        assert (infos[i].rows, infos[i].knees_found) == (inf1.rows, inf1.knees_found), i
        if st1 == OK:
            assert parts[i].tobytes() == pl1.tobytes(), i
    for i in (0, 7, 19):
        st_o, pl_o, info_o, _ = oracle.pack(sets[i])
        assert infos[i].scale_index == info_o.scale_index
        assert parts[i].tobytes() == np.ascontiguousarray(pl_o).tobytes(), i


def test_pack_many_device_pointers(ctx):
    import torch
    from paper_2602_07782_b200 import PLACEMENT_DTYPE, concat_chart_sets, spec_of
    sets = [chartgen.config5(i) for i in range(30, 38)]
    xy, cst, abase, res = concat_chart_sets(sets)
    st_h, pl_h, inf_h, ast_h, _ = ctx.pack_many(xy, cst, abase, spec_of(sets[0]), res_xy=res)
    st_d, out_d, inf_d, ast_d, bi = ctx.pack_many(torch.from_numpy(xy).cuda(),
                                                  torch.from_numpy(cst).cuda(), abase,
                                                  spec_of(sets[0]), res_xy=res)
    torch.cuda.synchronize()
    assert st_h == st_d and list(ast_h) == list(ast_d)
    assert [i.scale_index for i in inf_h] == [i.scale_index for i in inf_d]
    assert out_d.cpu().numpy().view(PLACEMENT_DTYPE).tobytes() == pl_h.tobytes()


def test_pack_many_edge_cases(orc):
    """Per-atlas status in one batch: a bad chart (EINVAL, atlas-local index),
    an atlas beyond the batch's 2,048-chart limit (packed solo), an atlas
    whose footprint slots overflow the batch's per-CTA buffers (grown,
    retried solo) -- and the good atlases around them unaffected; then an
    atlas where no scale fits (NO_FIT) beside one that fits."""
    import oracle
    from paper_2602_07782_b200 import (EINVAL, NO_FIT, OK, Context, concat_chart_sets,
                                       spec_of)
    ctx = Context(0, max_charts=4096, max_vertices=1 << 17, max_atlas_side=2048)
    good = chartgen.small_case(3, n=50, side=2048, family="tss", rho=0.8)
    bad = chartgen.from_polygons([[(0, 0), (9, 0), (9, 9), (0, 9)], [(0, 0), (5, 0), (0, 0)],
                                  [(1, 1), (4, 1), (4, 6)]], 2048, 2048)
    big = chartgen.generate("tss", 2300, 2048, 2048, 5, rho=0.7, side_limit=512)
    wide = chartgen.from_polygons([[(0, 0), (2000, 0), (2000, 2010), (0, 2010)]] * 10 +
                                  [[(0, 0), (40, 0), (40, 50), (0, 50)]] * 3, 2048, 2048)
    sets = [good, bad, big, wide, good]
    xy, cst, abase, res = concat_chart_sets(sets)
    st, pl, infos, ast, bi = ctx.pack_many(xy, cst, abase, spec_of(good), res_xy=res,
                                           raise_on_error=False)
    assert st == EINVAL
    assert list(ast) == [OK, EINVAL, OK, OK, OK]
    assert infos[1].bad_chart == 1
    assert bi.solo_atlases == 2  # big (> 2048 charts) and wide (capacity retry)
    parts = _split(pl, abase)
    for i in (0, 2, 3, 4):
        st1, pl1, inf1 = ctx.pack(sets[i].xy, sets[i].start, spec_of(sets[i]))
        assert st1 == OK and infos[i].scale_index == inf1.scale_index, i
        assert parts[i].tobytes() == pl1.tobytes(), i
    st_o, pl_o, info_o, _ = oracle.pack(wide)
    assert parts[3].tobytes() == np.ascontiguousarray(pl_o).tobytes()
    # a second batch on the grown workspace: the wide atlas now batches
    st, pl, infos, ast, bi = ctx.pack_many(xy, cst, abase, spec_of(good), res_xy=res,
                                           raise_on_error=False)
    assert list(ast) == [OK, EINVAL, OK, OK, OK] and bi.solo_atlases == 1
    assert _split(pl, abase)[3].tobytes() == np.ascontiguousarray(pl_o).tobytes()
    # NO_FIT: a 10,000-texel-wide chart in 64^2 does not fit even at 1/64
    fit = chartgen.from_polygons([[(0, 0), (10, 0), (10, 10), (0, 10)]], 64, 64)
    nofit = chartgen.from_polygons([[(0, 0), (10000, 0), (10000, 1), (0, 1)]], 64, 64)
    xy, cst, abase, res = concat_chart_sets([nofit, fit])
    st, pl, infos, ast, bi = ctx.pack_many(xy, cst, abase, spec_of(fit), res_xy=res)
    assert st == OK and list(ast) == [NO_FIT, OK]
    assert infos[0].scale_index == 0 and infos[1].scale_index == 64
    # area bound: m^2 * 10,000 <= 64^2 * 64^2 -> m_hi = 40, every one evaluated and failed
    # (a two-atlas batch runs several ranks per atlas at once: the fit atlas's
    # speculative ranks below its winner may be evaluated too)
    assert bi.candidates_evaluated >= 40 + 1
    ctx.close()


def test_pack_many_hybrid_spec_goes_solo(ctx):
    """t_opt > 0 (hybrid tail) is not batched: every atlas is packed by
    tabi_pack, with the same results."""
    from paper_2602_07782_b200 import concat_chart_sets, spec_of
    sets = [chartgen.config5(i) for i in range(3)]
    xy, cst, abase, res = concat_chart_sets(sets)
    spec = spec_of(sets[0], t_opt_bp=300)
    st, pl, infos, ast, bi = ctx.pack_many(xy, cst, abase, spec, res_xy=res)
    assert bi.batched_atlases == 0 and bi.solo_atlases == 3
    for i, (cs, part) in enumerate(zip(sets, _split(pl, abase))):
        st1, pl1, inf1 = ctx.pack(cs.xy, cs.start, spec)
        assert infos[i].scale_index == inf1.scale_index and part.tobytes() == pl1.tobytes()


def test_pack_many_deterministic_100_runs(ctx):
    """The queue's interleaving differs run to run; the bytes may not."""
    from paper_2602_07782_b200 import concat_chart_sets, spec_of
    sets = [chartgen.config5(i) for i in range(40, 56)]
    xy, cst, abase, res = concat_chart_sets(sets)
    ref = ctx.pack_many(xy, cst, abase, spec_of(sets[0]), res_xy=res)[1].tobytes()
    for _ in range(99):
        assert ctx.pack_many(xy, cst, abase, spec_of(sets[0]), res_xy=res)[1].tobytes() == ref


def test_single_pack_deterministic_100_runs(ctx):
    """100 packs of C3 at rho = 2.0 (fused kernel: the
    raster/packer handshake, early exit and tile queue all race) give one
    byte string."""
    from paper_2602_07782_b200 import spec_of
    cs = chartgen.config3(1, rho=2.0)
    ref = ctx.pack(cs.xy, cs.start, spec_of(cs))[1].tobytes()
    for _ in range(99):
        assert ctx.pack(cs.xy, cs.start, spec_of(cs))[1].tobytes() == ref


def test_pack_batch_uses_many(ctx):
    """tabi_pack_batch (one host thread per context) groups each context's
    atlases into one tabi_pack_many; results equal single packs."""
    from paper_2602_07782_b200 import Context, OK, pack_batch, spec_of
    sets = [chartgen.config5(i) for i in range(60, 70)]
    c2 = Context(0, max_charts=2100, max_vertices=1 << 17, max_atlas_side=2048)
    c3 = Context(0, max_charts=2100, max_vertices=1 << 17, max_atlas_side=2048)
    st, outs, infos = pack_batch([c2, c3], sets, [spec_of(cs) for cs in sets])
    assert st == OK
    for cs, pl, inf in zip(sets, outs, infos):
        st1, pl1, inf1 = ctx.pack(cs.xy, cs.start, spec_of(cs))
        assert inf.scale_index == inf1.scale_index and pl.tobytes() == pl1.tobytes()
    c2.close()
    c3.close()


@pytest.mark.parametrize("mode", [{"TABI_LAZY": "0"}, {"TABI_EARLY_FAIL": "0"}])
def test_pack_many_lazy_and_early_fail_are_exact(ctx, monkeypatch, mode):
    """The batch kernel's lazy raster and its row-end area test (R8)
    only skip work of candidates that fail: switching either off gives the
    same bytes on 48 C5 atlases (whose searches evaluate ~8 candidates each)."""
    from paper_2602_07782_b200 import concat_chart_sets, spec_of
    sets = [chartgen.config5(i) for i in range(100, 148)]
    xy, cst, abase, res = concat_chart_sets(sets)
    # one rank per atlas in flight: the evaluated-candidate count is then
    # schedule-independent (speculative ranks are compared below)
    monkeypatch.setenv("TABI_MANY_INFLIGHT", "1")
    monkeypatch.setenv("TABI_MANY_SPEC", "0")  # (no idle speculation either)
    ref = ctx.pack_many(xy, cst, abase, spec_of(sets[0]), res_xy=res)
    for k, v in mode.items():
        monkeypatch.setenv(k, v)
    alt = ctx.pack_many(xy, cst, abase, spec_of(sets[0]), res_xy=res)
    assert list(ref[3]) == list(alt[3])
    assert [i.scale_index for i in ref[2]] == [i.scale_index for i in alt[2]]
    assert ref[1].tobytes() == alt[1].tobytes()
    assert ref[4].candidates_evaluated == alt[4].candidates_evaluated


def test_pack_many_host_pinned_chunked_upload(ctx):
    """Host-pointer batch from pinned memory, large enough for the chunked
    outline upload (8 chunks on a copy stream, each chunk's proxies behind its
    copy): the same bytes as the device-pointer batch, with one chunk, and
    from pageable host buffers."""
    import torch
    from paper_2602_07782_b200 import OK, PLACEMENT_DTYPE, concat_chart_sets, spec_of
    sets = [chartgen.config5(i) for i in range(24)]
    xy, cst, abase, res = concat_chart_sets(sets)
    assert abase[-1] >= 8 * 2048
    st_d, out_d, _, ast_d, _ = ctx.pack_many(torch.from_numpy(xy).cuda(),
                                             torch.from_numpy(cst).cuda(), abase,
                                             spec_of(sets[0]), res_xy=res)
    torch.cuda.synchronize()
    ref = out_d.cpu().numpy().tobytes()
    xy_p = torch.from_numpy(xy).pin_memory().numpy()
    cst_p = torch.from_numpy(cst).pin_memory().numpy()
    out_p = torch.empty(int(abase[-1]) * 32, dtype=torch.uint8).pin_memory().numpy().view(PLACEMENT_DTYPE)
    for _ in range(2):
        out_p[:] = np.zeros(1, dtype=PLACEMENT_DTYPE)
        st, pl, _, ast, _ = ctx.pack_many(xy_p, cst_p, abase, spec_of(sets[0]), res_xy=res, out=out_p)
        assert st == st_d == OK and list(ast) == list(ast_d)
        assert pl.tobytes() == ref
    st, pl, _, ast, _ = ctx.pack_many(xy, cst, abase, spec_of(sets[0]), res_xy=res)  # pageable
    assert pl.tobytes() == ref


def test_pack_many_one_upload_chunk(ctx, monkeypatch):
    from paper_2602_07782_b200 import concat_chart_sets, spec_of
    sets = [chartgen.config5(i) for i in range(24)]
    xy, cst, abase, res = concat_chart_sets(sets)
    _, a, _, _, _ = ctx.pack_many(xy, cst, abase, spec_of(sets[0]), res_xy=res)
    monkeypatch.setenv("TABI_UPLOAD_CHUNKS", "1")
    _, b, _, _, _ = ctx.pack_many(xy, cst, abase, spec_of(sets[0]), res_xy=res)
    assert a.tobytes() == b.tobytes()


@pytest.mark.parametrize("k", ["1", "2", "8"])
def test_pack_many_ranks_in_flight_are_exact(ctx, monkeypatch, k):
    """Several ranks of one atlas in flight (speculative lower scales, the
    winner the lowest successful rank whose lower ranks all failed) give the
    bytes of the one-rank top-down search, on a small batch where the default
    runs 8 ranks per atlas and on a mix of NO_FIT and trivial atlases."""
    from paper_2602_07782_b200 import concat_chart_sets, spec_of
    sets = [chartgen.config5(i) for i in range(200, 212)] + \
        [chartgen.small_case(s, n=90, side=2048, family="tss", rho=3.0) for s in range(3)]
    xy, cst, abase, res = concat_chart_sets(sets)
    monkeypatch.setenv("TABI_MANY_INFLIGHT", "1")
    monkeypatch.setenv("TABI_MANY_SPEC", "0")
    ref = ctx.pack_many(xy, cst, abase, spec_of(sets[0]), res_xy=res, raise_on_error=False)
    monkeypatch.delenv("TABI_MANY_SPEC")
    monkeypatch.setenv("TABI_MANY_INFLIGHT", k)
    for carry in ("0", "1"):
        monkeypatch.setenv("TABI_MANY_CARRY", carry)
        for _ in range(3):
            alt = ctx.pack_many(xy, cst, abase, spec_of(sets[0]), res_xy=res, raise_on_error=False)
            assert list(ref[3]) == list(alt[3])
            assert [i.scale_index for i in ref[2]] == [i.scale_index for i in alt[2]]
            assert ref[1].tobytes() == alt[1].tobytes()


@pytest.mark.parametrize("spec", ["2", "3", "8"])
def test_pack_many_idle_speculation_is_exact(ctx, monkeypatch, spec):
    """Idle speculation (batch kernel): a CTA with no queued item
    starts the next rank of an undecided atlas, up to `spec` ranks in flight.
    One rank per atlas queued and far fewer atlases than CTAs, so almost every
    CTA speculates from the start -- on C5 atlases, NO_FIT atlases (every rank
    fails: the last outstanding rank, possibly a speculative index past the
    last candidate, decides them) and trivial ones; the bytes of the plain
    top-down search, run after run."""
    from paper_2602_07782_b200 import concat_chart_sets, spec_of
    from paper_2602_07782_b200 import NO_FIT
    # a 20,000 x 5 texel sliver exceeds the 2048^2 atlas at every scale m / 8:
    # all 8 ranks fail
    sliver = chartgen.from_polygons([[(0, 0), (20000, 0), (20000, 5), (0, 5)],
                                     [(0, 0), (30, 0), (30, 30), (0, 30)]], 2048, 2048)
    sets = [chartgen.config5(i) for i in range(300, 316)] + [sliver, sliver] + \
        [chartgen.small_case(s, n=90, side=2048, family="tss", rho=3.0) for s in range(3)] + \
        [chartgen.small_case(s, n=40, side=2048, family="tss", rho=0.2) for s in range(2)]
    xy, cst, abase, res = concat_chart_sets(sets)
    sp = spec_of(sets[0], scale_count=8)
    monkeypatch.setenv("TABI_MANY_INFLIGHT", "1")
    monkeypatch.setenv("TABI_MANY_SPEC", "0")
    ref = ctx.pack_many(xy, cst, abase, sp, res_xy=res, raise_on_error=False)
    assert list(ref[3][16:18]) == [NO_FIT, NO_FIT] and all(s == 0 for s in ref[3][:16])
    monkeypatch.setenv("TABI_MANY_SPEC", spec)
    for _ in range(4):
        alt = ctx.pack_many(xy, cst, abase, sp, res_xy=res, raise_on_error=False)
        assert list(ref[3]) == list(alt[3])
        assert [i.scale_index for i in ref[2]] == [i.scale_index for i in alt[2]]
        assert ref[1].tobytes() == alt[1].tobytes()
        assert alt[4].candidates_evaluated >= ref[4].candidates_evaluated
