"""Bit determinism of the CUDA path under repetition and schedule changes.

The fused wave kernel hands tiles between CTAs through release/acquire flags
and the batch kernel draws (atlas, candidate) items from a device queue, so
the order in which CTAs run differs from call to call.  The method's result
must not (P:85 / P:1025: one overlap-free packing per input; BASELINE
north_star: "deterministic tie-breaking").  compute-sanitizer is not
available on the GPU pool (DESIGN.md §6 "Race evidence"), so races are hunted
by repetition here: 100 packs of C3 at rho = 2.0 (the knee-rich case, several
candidates per wave) must return identical bytes, the same bytes as the split
(non-fused) path and as one-candidate waves, and a batch must be identical
across repeated calls.
"""
import numpy as np
import pytest

import chartgen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c3():
    return chartgen.config3(1, rho=2.0)


@pytest.fixture(scope="module")
def ctx():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    from paper_2602_07782_b200 import Context
    c = Context(0, max_charts=25000, max_vertices=1 << 19, max_atlas_side=8192)
    yield c
    c.close()


def _packs(ctx, cs, reps):
    import torch
    from paper_2602_07782_b200 import OK, spec_of
    xy = torch.from_numpy(cs.xy).cuda()
    st = torch.from_numpy(cs.start).cuda()
    outs = set()
    infos = set()
    for _ in range(reps):
        s, pl, info = ctx.pack(xy, st, spec_of(cs))
        assert s == OK
        outs.add(pl.cpu().numpy().tobytes() if hasattr(pl, "cpu") else np.asarray(pl).tobytes())
        infos.add((info.scale_index, info.rows, info.knees_found, info.knee_rows))
    return outs, infos


def test_hundred_packs_bit_identical(ctx, c3):
    outs, infos = _packs(ctx, c3, 100)
    assert len(outs) == 1 and len(infos) == 1


@pytest.mark.parametrize("env", [{"TABI_FUSED": "0"}, {"TABI_WAVE": "1"}, {"TABI_WAVE": "3"}])
def test_schedules_agree(ctx, c3, env, monkeypatch):
    ref, ref_info = _packs(ctx, c3, 1)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    outs, infos = _packs(ctx, c3, 10)
    assert outs == ref and infos == ref_info


def test_batch_repeats_bit_identical(ctx):
    import torch
    from paper_2602_07782_b200 import concat_chart_sets, spec_of
    sets = [chartgen.config5(i) for i in range(0, 96, 3)]
    xy, cst, abase, res = concat_chart_sets(sets)
    xy_d, cst_d = torch.from_numpy(xy).cuda(), torch.from_numpy(cst).cuda()
    seen = set()
    for _ in range(10):
        st, pl, infos, ast, bi = ctx.pack_many(xy_d, cst_d, abase, spec_of(sets[0]), res_xy=res)
        pb = pl.cpu().numpy().tobytes() if hasattr(pl, "cpu") else np.asarray(pl).tobytes()
        seen.add((pb, tuple(int(a) for a in ast), tuple(i.scale_index for i in infos)))
    assert len(seen) == 1
