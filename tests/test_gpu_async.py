"""The device-side candidate-wave loop and the asynchronous boundary
(tabi_pack_async / tabi_pack_query / tabi_pack_wait: "returns
after enqueueing, completion is stream-ordered").

The whole scale search is one CUDA graph: prologue, wave 0, a WHILE node whose
body is one further candidate wave, and the result copy; each wave's
select_kernel decides on the device whether another wave runs.  These tests
check that it gives the bytes of the host-driven loop (TABI_GRAPH=0) and of
the oracle, for one wave and for many (TABI_WAVE=1: one candidate per wave),
sequential and hybrid.
"""
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


CASES = [chartgen.config2(0), chartgen.config1b(3),
         chartgen.small_case(4, n=60, family="mixed", rho=1.3),
         chartgen.config3(2, rho=1.5)]


def _dev(cs):
    import torch
    return torch.from_numpy(cs.xy).cuda(), torch.from_numpy(cs.start).cuda()


@pytest.mark.parametrize("wave", ["16", "1"])
@pytest.mark.parametrize("cs", CASES, ids=lambda c: c.name)
def test_device_loop_equals_host_loop_and_oracle(ctx, cs, wave, monkeypatch):
    """Same placements and statistics from the graph's device-side wave loop
    and the host-driven loop; the winner is the oracle's.  With one candidate
    per wave the device loop runs many waves inside one graph launch."""
    import oracle
    from paper_2602_07782_b200 import spec_of
    monkeypatch.setenv("TABI_WAVE", wave)
    spec = spec_of(cs)
    st_d, pl_d, info_d = ctx.pack(cs.xy, cs.start, spec)
    monkeypatch.setenv("TABI_GRAPH", "0")
    st_h, pl_h, info_h = ctx.pack(cs.xy, cs.start, spec)
    monkeypatch.delenv("TABI_GRAPH")
    assert st_d == st_h
    assert pl_d.tobytes() == pl_h.tobytes()
    assert (info_d.scale_index, info_d.rows, info_d.knees_found, info_d.knee_rows) == (
        info_h.scale_index, info_h.rows, info_h.knees_found, info_h.knee_rows)
    assert info_d.gpu_launches == info_h.gpu_launches  # same kernels, waves decided on the device
    st_o, pl_o, info_o, _ = oracle.pack(cs, with_cands=True)
    assert st_d == st_o and info_d.scale_index == info_o.scale_index
    assert pl_d.tobytes() == np.ascontiguousarray(pl_o).tobytes()


def test_device_loop_hybrid_tail(ctx, monkeypatch):
    """Hybrid mode (D25): the device loop continues past a success while a lower
    candidate could still have a larger area-weighted scale."""
    import oracle
    from paper_2602_07782_b200 import spec_of
    cs = chartgen.small_case(2, n=300, family="lightmap", side=1024, rho=0.8)
    for wave in ("16", "2"):
        monkeypatch.setenv("TABI_WAVE", wave)
        st_d, pl_d, info_d = ctx.pack(cs.xy, cs.start, spec_of(cs, t_opt_bp=300))
        monkeypatch.setenv("TABI_GRAPH", "0")
        st_h, pl_h, info_h = ctx.pack(cs.xy, cs.start, spec_of(cs, t_opt_bp=300))
        monkeypatch.delenv("TABI_GRAPH")
        assert st_d == st_h and pl_d.tobytes() == pl_h.tobytes()
        assert info_d.l2_stretch == info_h.l2_stretch
    st_o, pl_o, info_o, _ = oracle.pack(cs, with_cands=True, t_opt_bp=300)
    assert info_d.scale_index == info_o.scale_index
    assert pl_d.tobytes() == np.ascontiguousarray(pl_o).tobytes()


def test_async_equals_sync(ctx):
    """tabi_pack_async returns after enqueueing; tabi_pack_wait then gives the
    status, info and placements of a synchronous device-pointer pack."""
    import torch
    from paper_2602_07782_b200 import OK, PENDING, PLACEMENT_DTYPE, spec_of
    for cs in CASES:
        xy, start = _dev(cs)
        st_s, out_s, info_s = ctx.pack(xy, start, spec_of(cs))
        torch.cuda.synchronize()
        out = ctx.pack_async(xy, start, spec_of(cs))
        q = ctx.query()
        assert q in (OK, PENDING)
        st, out2, info = ctx.wait()
        assert out2 is out
        assert st == st_s == OK
        assert (info.scale_index, info.rows, info.knees_found, info.gpu_launches) == (
            info_s.scale_index, info_s.rows, info_s.knees_found, info_s.gpu_launches)
        assert info.l2_stretch == info_s.l2_stretch
        torch.cuda.synchronize()
        assert out.cpu().numpy().tobytes() == out_s.cpu().numpy().tobytes()
        assert out.cpu().numpy().view(PLACEMENT_DTYPE).shape[0] == cs.n_charts


def test_async_overlaps_host_work_and_rejects_misuse(ctx):
    """While a pack is in flight: a second enqueue or a synchronous pack on the
    same context is refused (EINVAL), query() never blocks; wait() twice is
    EINVAL the second time."""
    from paper_2602_07782_b200 import EINVAL, OK, PENDING, TabiError, spec_of
    cs = chartgen.config3(0, rho=1.5)
    xy, start = _dev(cs)
    ctx.pack_async(xy, start, spec_of(cs))
    with pytest.raises(TabiError) as e:
        ctx.pack_async(xy, start, spec_of(cs))
    assert e.value.status == EINVAL
    st, _, _ = ctx.pack(xy, start, spec_of(cs), raise_on_error=False)
    assert st == EINVAL
    seen = set()
    for _ in range(100000):
        q = ctx.query()
        seen.add(q)
        if q == OK:
            break
    assert seen <= {OK, PENDING} and OK in seen
    st, _, info = ctx.wait()
    assert st == OK and info.scale_index > 0
    st, _, _ = ctx.wait(raise_on_error=False)
    assert st == EINVAL


def test_async_capacity_growth_and_errors():
    """A fresh context whose footprint buffers are too small: the device-side
    check stops the graph, tabi_pack_wait grows them and re-runs -- same bytes
    as a synchronous pack.  An invalid chart is reported by wait()."""
    import torch
    from paper_2602_07782_b200 import Context, EINVAL, OK, spec_of
    cs = chartgen.config3(1, rho=2.0)
    xy, start = _dev(cs)
    ref = Context(0, max_charts=cs.n_charts, max_vertices=cs.n_vertices, max_atlas_side=4096)
    st_r, out_r, info_r = ref.pack(xy, start, spec_of(cs))
    torch.cuda.synchronize()
    c = Context(0, max_charts=cs.n_charts, max_vertices=cs.n_vertices, max_atlas_side=4096)
    out = c.pack_async(xy, start, spec_of(cs))
    st, _, info = c.wait()
    torch.cuda.synchronize()
    assert st == st_r == OK and info.scale_index == info_r.scale_index
    assert out.cpu().numpy().tobytes() == out_r.cpu().numpy().tobytes()
    # a degenerate chart: found on the device, reported at wait()
    bad = cs.xy.copy()
    s0, s1 = int(cs.start[5]), int(cs.start[6])
    bad[2 * s0:2 * s1] = 0.0
    c.pack_async(torch.from_numpy(bad).cuda(), start, spec_of(cs))
    st, _, info = c.wait(raise_on_error=False)
    assert st == EINVAL and info.bad_chart == 5
    c.close()
    ref.close()


def test_new_device_pointers_update_the_graph(ctx):
    """Device-pointer packs whose buffers move between calls (same sizes and
    spec): the graph is re-captured and updated in place -- every call still
    reads its own inputs and writes its own output."""
    import torch
    from paper_2602_07782_b200 import OK, spec_of
    cs = chartgen.config2(3)
    ref = None
    for i in range(4):
        xy, start = _dev(cs)
        pad = torch.zeros(1024 * (i + 1), device="cuda")  # (moves later allocations)
        st, out, info = ctx.pack(xy, start, spec_of(cs))
        torch.cuda.synchronize()
        assert st == OK
        b = out.cpu().numpy().tobytes()
        ref = ref or b
        assert b == ref
        del pad
    # another chart set with the same chart count (other vertex count): the
    # updated graph must read the new buffers, not the previous call's
    cs2 = chartgen.config2(4)
    assert cs2.n_charts == cs.n_charts
    xy2, start2 = _dev(cs2)
    st, out2, _ = ctx.pack(xy2, start2, spec_of(cs2))
    st_h, pl_h, _ = ctx.pack(cs2.xy, cs2.start, spec_of(cs2))
    torch.cuda.synchronize()
    assert st == st_h == OK
    assert out2.cpu().numpy().tobytes() == pl_h.tobytes()
