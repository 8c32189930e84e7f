#!/usr/bin/env python
"""Benchmark of the B200-native TABI packer (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload C3|C2|C4] [--rho R]

A *step* is one full pack (all five hot-path stages, all 64 candidate scales)
of one synthetic chart set of the metric's workload (configs[2]: 1,572 TSS-like
charts into a 4096^2 atlas, k = 10, t_opt = 0) with inputs resident in HBM.
Each rank packs its own atlas per step (seed = rank): weak scaling, no data-path
collective; value = atlases/s over all ranks = N*K / max-over-
ranks device time.  L2 is flushed (256 MB write) between steps, outside the
timed events.  Device time per step = the CUDA-event span tabi_pack records on
the timed stream around its own enqueued work (tabi_info.device_ms); the
outer per-step events (which also see the host return from the synchronous
call) are reported as stream_ms_per_step.  Everything timed runs on one
dedicated stream, so the flush is complete before a pack starts.  `e2e` repeats the measurement through the public host-pointer
call (H2D of the chart set and D2H of the placements inside the timed region).
`--impl reference` times the CPU oracle (the only reference this paper has:
no code) on the box's host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "p50 pack ms @1572 charts 4096² atlas; L2 stretch; atlases/s at 1/2/4/8 B200"
PAPER_CONTEXT = ("paper (RTX 4090, OpenGL): 5.31 ms mean pack for 1,001-5,000 charts (P:672), "
                 "15 ms interactive budget (P:35); Xatlas-random >= 2.5 s for 1,572 charts on a "
                 "Ryzen 7 1800X (P:39)")


# spec overrides per workload (beyond the chart set's own fields)
WORKLOAD_SPEC = {"C4X": {"flags": 32}}


def workload(name: str, seed: int, rho: float):
    import chartgen
    if name == "C3":
        cs = chartgen.config3(seed, rho=rho)
        desc = (f"C3 configs[2]: 1572 tss charts (chartgen seed={seed}, rho={rho}) into 4096x4096, "
                f"k=10, t_opt=0, M=64, gutter=1")
    elif name == "C2":
        cs = chartgen.config2(seed)
        desc = f"C2 configs[1]: 214 uv charts (seed={seed}, rho=1.1) into 1024x1024, k=10, M=64, g=1"
    elif name == "C4":
        cs = chartgen.config4(seed, t_opt_bp=0)
        desc = f"C4 configs[3]: 20000 lightmap charts (seed={seed}, rho=0.8) into 8192x8192, t_opt=0"
    elif name == "C4X":
        cs = chartgen.config4(seed, t_opt_bp=-1)
        desc = (f"C4 configs[3]: 20000 lightmap charts (seed={seed}, rho=0.8) into 8192x8192, "
                f"paper t_opt policy with the exact-greedy tail (TABI_F_EXACT_TAIL, SURVEY N4)")
    elif name == "C4P":
        cs = chartgen.config4(seed, t_opt_bp=-1)
        desc = (f"C4 configs[3]: 20000 lightmap charts (seed={seed}, rho=0.8) into 8192x8192, "
                f"paper t_opt policy (1% for > 10,000 charts, hybrid prefix tail)")
    else:
        raise SystemExit(f"unknown workload {name}")
    return cs, desc


class ClockSampler:
    """nvidia-smi-equivalent clocks / throttle reasons sampled via NVML during the timed region."""

    REASONS = {"gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
               "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
               "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80}

    def __init__(self, device: int):
        self.samples, self.reasons, self.max_mhz = [], 0, None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        names = [k for k, v in self.REASONS.items() if self.reasons & v and k != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": names, "samples": len(self.samples)}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured"
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


def dist_setup():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist
        import torch
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return ws, rank, local


def allmax(x: float, ws: int) -> float:
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def cpu_oracle_rate(cs, budget_s=15.0, max_candidates=None, **spec_kw):
    """Time the oracle (as it stands) on host cores: full packs until ~budget_s."""
    import oracle
    oracle.build()
    t0 = time.perf_counter()
    n = 0
    while True:
        st, pl, info, _ = oracle.pack(cs, **spec_kw)
        n += 1
        if time.perf_counter() - t0 > budget_s or n >= 64:
            break
    dt = time.perf_counter() - t0
    return n / dt, n, dt, info.scale_index


def run_reference(args, ws, rank):
    if rank != 0:
        return
    import oracle
    oracle.build()
    cs, desc = workload(args.workload, 0, args.rho)
    kw = WORKLOAD_SPEC.get(args.workload, {})
    sample_cands = args.steps > 20
    M = cs.scale_count

    def step(i):
        if not sample_cands:
            t = time.perf_counter()
            oracle.pack(cs, **kw)
            return time.perf_counter() - t
        # bounded sample: proxies+sort+8 of the 64 candidate scales (rotating), scaled to 64
        ms = [M - ((i % 8) + 8 * j) for j in range(8)]
        t = time.perf_counter()
        for m in ms:
            oracle.pack_candidate(cs, m, **kw)
        return (time.perf_counter() - t) * M / len(ms)

    for i in range(args.warmup):
        step(i)
    times = [step(i) for i in range(args.steps)]
    ms_step = 1000.0 * sum(times) / len(times)
    value = 1000.0 / ms_step
    sample = ("one full oracle pack per step (all 64 candidates)" if not sample_cands else
              "per step: 8 of the 64 candidate scales (rotating) + proxies/sort, time x 8")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "atlases/s",
            "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
            "data": "synthetic (chartgen, SplitMix64)",
            "config": {"workload": desc, "impl": "CPU oracle (oracle/, plain C, 1 thread)"},
            "p50_ms": 1000.0 * statistics.median(times),
            "cpu_baseline": {"value": value, "unit": "atlases/s", "cores": 1, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": "atlases/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def rank_atlases(name, rank, ws, rho):
    """The chart sets this rank packs each step, and the per-step total over ranks."""
    if name == "C5":
        import chartgen
        from paper_2602_07782_b200 import shard_plan
        sizes = chartgen.config5_sizes(512)
        a = shard_plan(sizes, ws)
        mine = [chartgen.config5(i) for i in range(512) if a[i] == rank]
        desc = ("C5 configs[4]: batch of 512 tss atlases (200-2000 charts each, rho~U[0.3,1.5]) "
                "into 2048x2048, LPT-sharded over the ranks")
        return mine, desc, 512, "strong"
    cs, desc = workload(name, rank, rho)
    return [cs], desc, ws, "weak"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="C3")
    ap.add_argument("--rho", type=float, default=0.5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--flush", default="write", choices=["write", "write+read", "none"],
                    help="L2 flush between timed steps: a 256 MB write (default), or that "
                         "write followed by a 256 MB read so L2 holds no dirty lines; "
                         "'none' is a warm-cache diagnostic, not a bench value")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    ws, rank, local = dist_setup()
    if args.impl == "reference":
        run_reference(args, ws, rank)
        return

    import numpy as np
    import torch

    from paper_2602_07782_b200 import Context, spec_of
    from paper_2602_07782_b200 import build as nbuild
    if nbuild.needs_build():
        nbuild.build()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    sets, desc, units_per_step, scaling = rank_atlases(args.workload, rank, ws, args.rho)
    specs = [spec_of(cs, **WORKLOAD_SPEC.get(args.workload, {})) for cs in sets]
    ctx = Context(local, max_charts=max(max(cs.n_charts for cs in sets), 1024),
                  max_vertices=max(cs.n_vertices for cs in sets) + 16,
                  max_atlas_side=max(max(cs.atlas_w, cs.atlas_h) for cs in sets))
    # one dedicated stream for everything timed: the L2 flush, the CUDA events and
    # the packs (torch's default stream is the legacy NULL stream, handle 0,
    # which the C ABI would read as "the context's own stream")
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    dev_in = [(torch.from_numpy(cs.xy).to(dev), torch.from_numpy(cs.start).to(dev),
               torch.empty(cs.n_charts * 32, dtype=torch.uint8, device=dev)) for cs in sets]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    flush_rd = torch.zeros(64 << 20, dtype=torch.int32, device=dev) if args.flush == "write+read" \
        else None

    def do_flush():
        if args.flush == "none":
            return
        flush.zero_()
        if flush_rd is not None:
            flush_rd.sum()

    def step_dev():
        infos = []
        for (xy_d, start_d, out_d), spec in zip(dev_in, specs):
            infos.append(ctx.pack(xy_d, start_d, spec, out=out_d, stream=stream.cuda_stream)[2])
        return infos

    os.environ["TABI_TIMING"] = "0"
    for _ in range(args.warmup):
        step_dev()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    launches = 0
    work_pack = work_prof = 0
    infos = None
    span_ms = []  # per step: the library's own device span (tabi_info.device_ms)
    barrier(ws)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            do_flush()
            ev[i][0].record(stream)
            infos = step_dev()
            ev[i][1].record(stream)
            span_ms.append(sum(info.device_ms for info in infos))
            for info in infos:
                launches += info.gpu_launches
                work_pack += info.work_pack
                work_prof += info.work_profile
    torch.cuda.synchronize()
    barrier(ws)
    # per-stage device times (TABI_TIMING events inside tabi_pack) from separate,
    # untimed steps: the events and their host syncs stay out of the timed loop
    os.environ["TABI_TIMING"] = "1"
    stage = np.zeros(8)
    stage_steps = min(args.steps, 20)
    for i in range(stage_steps):
        do_flush()
        for info in step_dev():
            stage += np.array(info.stage_ms[:8])
    torch.cuda.synchronize()
    os.environ["TABI_TIMING"] = "0"
    # device time per step = the pack's own span on the timed stream (CUDA events
    # recorded by tabi_pack around its enqueued work, tabi_info.device_ms); the
    # outer events bracketing each step additionally see the host returning from
    # the synchronous call (reported as stream_ms_per_step)
    outer_ms = [a.elapsed_time(b) for a, b in ev]
    step_ms = span_ms
    total_ms = allmax(sum(step_ms), ws)
    outer_total = allmax(sum(outer_ms), ws)
    ms_per_step = total_ms / args.steps
    value = units_per_step * args.steps / (total_ms / 1000.0)
    p50 = statistics.median(step_ms)
    p99 = float(np.percentile(step_ms, 99))

    # ---- e2e through the public host-pointer call -------------------------
    e2e_steps = max(10, args.steps // 4) if len(sets) == 1 else 3
    for cs, spec in zip(sets, specs):
        ctx.pack(cs.xy, cs.start, spec, stream=stream.cuda_stream)
    e2e_ev = []
    torch.cuda.synchronize()
    barrier(ws)
    for i in range(e2e_steps):
        do_flush()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for cs, spec in zip(sets, specs):
            ctx.pack(cs.xy, cs.start, spec, stream=stream.cuda_stream)
        b.record(stream)
        e2e_ev.append((a, b))
    torch.cuda.synchronize()
    e2e_ms = allmax(sum(a.elapsed_time(b) for a, b in e2e_ev), ws) / e2e_steps
    h2d = int(sum(cs.xy.nbytes + cs.start.nbytes for cs in sets))
    d2h = int(sum(cs.n_charts * 32 + 64 + 56 * cs.scale_count for cs in sets))

    # ---- roofline of the dominant kernel -------------------------------
    npk = args.steps * len(sets)
    stage_avg = stage / (stage_steps * len(sets))
    names = ["h2d", "proxies", "sort", "profiles", "offsets_locks", "fold_push", "select", "d2h"]
    k_dom = int(np.argmax(stage_avg[1:7])) + 1
    pk, pk_kind = peaks()
    sm_mhz = pk.get("sm_max_mhz", 1965.0)
    # int32 lane-op issue peak: 148 SMs x 4 SMSPs x 32 lanes x clock
    alu_peak = 148 * 128 * sm_mhz * 1e6 / 1e9  # G lane-ops/s
    fused = bool(infos[0].fused)
    if fused and k_dom == 5:
        # the fused wave kernel rasterizes footprints (K3), computes pair offsets
        # (K3b) and runs the row loop (K4) in one launch: its work is both
        work = (work_pack + work_prof) / npk
        names[5] = "fused_wave (K3+K3b+K4)"
    else:
        work = {5: work_pack / npk, 3: work_prof / npk}.get(k_dom)
    roof = {"kernel": names[k_dom], "bound": "alu", "unit": "Gop/s",
            "peak": alu_peak, "peak_kind": f"derived from {pk_kind} sm_max_mhz (148x128 int32 lanes)",
            "stage_ms": {names[i]: round(float(stage_avg[i]), 5) for i in range(8)},
            "traffic": None}
    if work is not None and stage_avg[k_dom] > 0:
        ach = work / (stage_avg[k_dom] * 1e-3) / 1e9
        roof.update({"achieved": ach, "frac": ach / alu_peak,
                     "work_per_launch": work,
                     "work_unit": ("frontline column visits + footprint entries"
                                   if fused and k_dom == 5 else
                                   "frontline column visits" if k_dom == 5 else
                                   "footprint entries")})
    else:
        roof.update({"achieved": None, "frac": None})
    tr = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tr):
        roof["traffic"] = json.load(open(tr)).get(args.workload, {}).get(names[k_dom])
    # HBM context: compulsory bytes per pack
    hbm_bytes = sum(cs.xy.nbytes + cs.start.nbytes + 32 * cs.n_charts for cs in sets) / len(sets)
    info = infos[0]
    line = {"metric": METRIC, "value": value, "unit": "atlases/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "int32",
            "data": "synthetic (chartgen SplitMix64, seed = rank)",
            "config": {"workload": desc,
                       "l2": {"write": "flushed between steps (256 MB write, untimed)",
                              "write+read": "flushed between steps (256 MB write + 256 MB read, "
                                            "untimed)",
                              "none": "NOT flushed (warm-cache diagnostic, not a bench value)"
                              }[args.flush],
                       "parallelism": (f"{ws} independent packs per step (one per GPU)"
                                       if scaling == "weak" else
                                       f"512 atlases per step sharded over {ws} GPU(s)")},
            "p50_ms": p50, "p99_ms": p99,
            "stream_ms_per_step": outer_total / args.steps,
            "l2_stretch": (info.l2_stretch if len(sets) == 1 else
                           float(np.mean([i.l2_stretch for i in infos]))),
            "scale_index": info.scale_index, "rows": info.rows,
            "interactive_budget_ms": 15.0,
            "hbm_compulsory": {"bytes_per_pack": int(hbm_bytes),
                               "gbs": hbm_bytes * len(sets) / (p50 * 1e-3) / 1e9,
                               "frac_of_measured": hbm_bytes * len(sets) / (p50 * 1e-3) / 1e9 /
                               pk.get("hbm_gbs", 6650.0)},
            "roofline": roof,
            "e2e": {"value": units_per_step * 1000.0 / e2e_ms, "unit": "atlases/s",
                    "ms_per_step": e2e_ms, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "paper_context": PAPER_CONTEXT}
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        rate, n, dt, m = cpu_oracle_rate(sets[0], **WORKLOAD_SPEC.get(args.workload, {}))
        line["cpu_baseline"] = {"value": rate, "unit": "atlases/s", "cores": 1, "kind": "oracle",
                                "sample": f"{n} full oracle packs of the first chart set "
                                          f"(all candidates) in {dt:.1f} s, 1 thread",
                                "host_cores": os.cpu_count()}
    if rank == 0:
        print(json.dumps(line))
    ctx.close()
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
