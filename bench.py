#!/usr/bin/env python
"""Benchmark of the B200-native TABI packer (BASELINE.json metric:
"p50 pack ms @1572 charts 4096^2 atlas; L2 stretch; atlases/s at 1/2/4/8 B200").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload C5|C3|C2|C4|C4P|C4X] [--rho R] [--quick]

Default (workload C5): the metric's throughput part, "atlases/s at 1/2/4/8
B200", on configs[4] -- a batch of 512 independent atlases (200-2,000 TSS-like
charts each, 2048^2) sharded over the ranks by LPT (strong scaling, no
data-path collective: SURVEY §8(e)).  A *step* packs every atlas of the rank's
share through ONE tabi_pack_many call (all hot-path stages for every atlas:
batched proxies, per-atlas sort, (atlas, candidate) work queue of raster +
pair offsets + Alg. 4, placements) with inputs resident in HBM.  value = 512 *
K / (max over ranks of the summed step times), step time = CUDA events on the
timed stream around the call.  L2 is flushed (256 MB write) between steps,
outside the events.  `e2e` repeats it through the host-pointer call from
pinned memory (H2D of the outlines and D2H of the placements inside the timed
region); `batch.wall_atlases_per_s` is the same call by the host wall clock.

At N = 1 the line also carries the metric's latency part on configs[2]
(1,572 charts into 4096^2, k = 10, t_opt = 0): p50 / p99 single-pack latency
(`tabi_pack`, device pointers, the pack's own CUDA-event span) over seeds 0-7 at
rho = 1.5 -- the fill ratio whose stretch (~1.39) matches the paper's 2K TSS
regime (1.38) -- and at rho = 0.5 / 2.0; a knob sweep k x t_opt
(P:897); the latency floor of the packer's building blocks; the
roofline of the dominant kernel; and the CPU oracle on the box's cores.

--workload C3|C2|C4|C4P|C4X: the round-1 single-pack bench (one atlas per
rank per step, weak scaling), kept for diagnostics.
`--impl reference` times the CPU oracle (the only reference this paper has --
no code) on the same workload, metric and unit, on the box's host cores.
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
C5_ATLASES = 512
C3_HEADLINE_RHO = 1.5

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


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


# ---------------------------------------------------------------- C5 batch --

def _gen_c5(i):
    import chartgen
    return chartgen.config5(i)


def c5_sets(indices, procs=None):
    """configs[4] atlases by index, generated in parallel (pure-Python generator)."""
    import multiprocessing as mp
    if len(indices) <= 4:
        return [_gen_c5(i) for i in indices]
    ctx = mp.get_context("fork")
    with ctx.Pool(procs or min(host_cores(), 32)) as pool:
        return pool.map(_gen_c5, indices, chunksize=4)


def rank_share(ws, rank):
    import chartgen
    from paper_2602_07782_b200 import shard_plan
    sizes = chartgen.config5_sizes(C5_ATLASES)
    a = shard_plan(sizes, ws)
    return [i for i in range(C5_ATLASES) if a[i] == rank]


def _oracle_pack_time(cs):
    import oracle
    t = time.perf_counter()
    st, pl, info, _ = oracle.pack(cs)
    return time.perf_counter() - t, info.scale_index


def oracle_batch_rate(sets, budget_s=12.0):
    """The oracle (as it stands, 1 thread per pack) on the box's host cores:
    one process per core, each packing whole atlases of `sets` (rotating) until
    ~budget_s.  Returns (atlases/s on all cores, atlases/s on one core, cores,
    atlases packed, wall seconds)."""
    import multiprocessing as mp
    import oracle
    oracle.build()
    cores = host_cores()
    ctx = mp.get_context("fork")
    done, t_sum = 0, 0.0
    t0 = time.perf_counter()
    with ctx.Pool(cores) as pool:
        i = 0
        while time.perf_counter() - t0 < budget_s and i < 4 * len(sets):
            chunk = [sets[(i + j) % len(sets)] for j in range(cores)]
            res = pool.map(_oracle_pack_time, chunk, chunksize=1)
            done += len(chunk)
            t_sum += sum(r[0] for r in res)
            i += cores
    wall = time.perf_counter() - t0
    return done / wall, done / t_sum, cores, done, wall


def run_reference(args, ws, rank):
    """--impl reference: the CPU oracle on the same workload / metric / unit.
    Rank 0 alone runs it under torchrun."""
    if rank != 0:
        return
    import oracle
    oracle.build()
    cores = host_cores()
    if args.workload == "C5":
        # a bounded, deterministic sample of the batch: every 8th atlas
        sets = c5_sets(list(range(0, C5_ATLASES, 8)))
        import multiprocessing as mp
        # atlases per step: all cores busy, whole run within a few minutes
        per = cores if args.steps <= 40 else max(1, cores * 40 // args.steps)
        pool = mp.get_context("fork").Pool(cores)

        def step(i):
            chunk = [sets[(i * per + j) % len(sets)] for j in range(per)]
            t = time.perf_counter()
            pool.map(_oracle_pack_time, chunk, chunksize=1)
            return time.perf_counter() - t, len(chunk)

        for i in range(args.warmup):
            step(i)
        rs = [step(args.warmup + i) for i in range(args.steps)]
        pool.close()
        tot_t = sum(r[0] for r in rs)
        tot_a = sum(r[1] for r in rs)
        value = tot_a / tot_t
        desc = ("C5 configs[4]: 512 tss atlases (200-2000 charts, 2048x2048); oracle sample "
                f"= every 8th atlas, {per} per step")
        sample = (f"per step: {per} whole C5 atlases (every 8th of the batch, rotating), one "
                  f"oracle pack (all 64 candidates) per process, {cores} processes")
        ms_step = 1000.0 * tot_t / len(rs)
    else:
        cs, desc = workload(args.workload, 0, args.rho)
        kw = WORKLOAD_SPEC.get(args.workload, {})

        def step(i):
            t = time.perf_counter()
            oracle.pack(cs, **kw)
            return time.perf_counter() - t

        for i in range(args.warmup):
            step(i)
        times = [step(i) for i in range(args.steps)]
        ms_step = 1000.0 * sum(times) / len(times)
        value = 1000.0 / ms_step
        cores = 1
        sample = "one full oracle pack per step (all 64 candidates), 1 thread"
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "atlases/s",
            "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong" if args.workload == "C5" else "weak",
            "vs_baseline": None, "dtype": "int64", "data": "synthetic (chartgen, SplitMix64)",
            "config": {"workload": desc, "impl": "CPU oracle (oracle/, plain C)"},
            "cpu_baseline": {"value": value, "unit": "atlases/s", "cores": cores, "kind": "oracle",
                             "sample": sample, "cpu_model": cpu_model()},
            "e2e": {"value": value, "unit": "atlases/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def c3_latency(ctx, stream, dev, rho, seeds, reps, flush):
    """tabi_pack latency (device pointers, the pack's own CUDA-event span) over
    seeds x reps, L2 flushed before each pack."""
    import torch
    from paper_2602_07782_b200 import spec_of
    ms, stretch, rows, ms_m = [], [], [], []
    for seed in seeds:
        cs, _ = workload("C3", seed, rho)
        xy = torch.from_numpy(cs.xy).to(dev)
        st = torch.from_numpy(cs.start).to(dev)
        out = torch.empty(cs.n_charts * 32, dtype=torch.uint8, device=dev)
        spec = spec_of(cs)
        for _ in range(3):
            ctx.pack(xy, st, spec, out=out, stream=stream.cuda_stream)
        for _ in range(reps):
            flush()
            info = ctx.pack(xy, st, spec, out=out, stream=stream.cuda_stream)[2]
            ms.append(info.device_ms)
        stretch.append(info.l2_stretch)
        rows.append(info.rows)
        ms_m.append(info.scale_index)
    ms.sort()
    p99 = ms[min(len(ms) - 1, int(round(0.99 * (len(ms) - 1))))]
    return {"rho": rho, "seeds": list(seeds), "packs": len(ms), "p50_ms": statistics.median(ms),
            "p99_ms": p99, "mean_ms": statistics.fmean(ms), "l2_stretch_mean": statistics.fmean(stretch),
            "l2_stretch": stretch, "scale_index": ms_m, "rows": rows}


def shard_shares(ctx, stream, dev, flush, spec, reps=3):
    """The per-GPU work of the multi-GPU C5 step, measured on this GPU: for
    N = 2, 4, 8 every rank's LPT share (the exact share bench.py --gpus N
    gives that rank) packed by one tabi_pack_many, device span median of
    `reps`.  The N-GPU step has no inter-GPU work (no data-path collective),
    so its time is the slowest share's: 512 / that time is what an N-GPU run
    of this build delivers on this GPU model (an N-GPU run measures it
    directly)."""
    import numpy as np
    import torch
    from paper_2602_07782_b200 import concat_chart_sets
    out = {}
    for n in (2, 4, 8):
        per = []
        for r in range(n):
            sets = c5_sets(rank_share(n, r))
            xy, cst, abase, res = concat_chart_sets(sets)
            xy_d, cst_d = torch.from_numpy(xy).to(dev), torch.from_numpy(cst).to(dev)
            ctx.pack_many(xy_d, cst_d, abase, spec, res_xy=res, stream=stream.cuda_stream)
            ts = []
            for _ in range(reps):
                flush()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                ctx.pack_many(xy_d, cst_d, abase, spec, res_xy=res, stream=stream.cuda_stream)
                b.record(stream)
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            per.append(float(np.median(ts)))
        out[f"gpus_{n}"] = {"share_ms": [round(x, 3) for x in per], "max_share_ms": max(per),
                            "atlases_per_s": C5_ATLASES * 1000.0 / max(per)}
    return out


def knob_sweep(ctx, stream, dev, flush, reps=8):
    """C3 (rho = 1.5, seed 0): local-AABB count k x t_opt."""
    import torch
    from paper_2602_07782_b200 import spec_of
    cs, _ = workload("C3", 0, C3_HEADLINE_RHO)
    xy = torch.from_numpy(cs.xy).to(dev)
    st = torch.from_numpy(cs.start).to(dev)
    out = torch.empty(cs.n_charts * 32, dtype=torch.uint8, device=dev)
    rows = []
    for k in (2, 5, 10):
        for t in (0, 100, 200, 500):
            spec = spec_of(cs, local_aabb_count=k, t_opt_bp=t)
            for _ in range(2):
                ctx.pack(xy, st, spec, out=out, stream=stream.cuda_stream)
            ms = []
            for _ in range(reps):
                flush()
                info = ctx.pack(xy, st, spec, out=out, stream=stream.cuda_stream)[2]
                ms.append(info.device_ms)
            rows.append({"k": k, "t_opt_pct": t / 100.0, "p50_ms": statistics.median(ms),
                         "l2_stretch": info.l2_stretch, "scale_index": info.scale_index,
                         "rows": info.rows, "prefix_rows": info.prefix_rows})
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="C5")
    ap.add_argument("--rho", type=float, default=C3_HEADLINE_RHO)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--quick", action="store_true", help="skip the C3 blocks and the knob sweep")
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
    if args.workload != "C5":
        run_single(args, ws, rank, local)
        return

    import numpy as np
    import torch

    from paper_2602_07782_b200 import Context, concat_chart_sets, latency_floor, spec_of
    from paper_2602_07782_b200 import build as nbuild
    if nbuild.needs_build():
        nbuild.build()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    share = rank_share(ws, rank)
    sets = c5_sets(share)
    xy, cst, abase, res = concat_chart_sets(sets)
    spec = spec_of(sets[0])
    N, V, A = int(abase[-1]), int(cst[-1]), len(sets)
    ctx = Context(local, max_charts=25000, max_vertices=1 << 19, max_atlas_side=4096)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    flush_rd = (torch.zeros(64 << 20, dtype=torch.int32, device=dev)
                if args.flush == "write+read" else None)

    def flush():
        if args.flush == "none":
            return
        flush_buf.zero_()
        if flush_rd is not None:
            flush_rd.sum()

    xy_d = torch.from_numpy(xy).to(dev)
    cst_d = torch.from_numpy(cst).to(dev)
    out_d = torch.empty(N * 32, dtype=torch.uint8, device=dev)
    os.environ["TABI_TIMING"] = "0"

    def step_dev():
        return ctx.pack_many(xy_d, cst_d, abase, spec, res_xy=res, out=out_d,
                             stream=stream.cuda_stream)

    for _ in range(args.warmup):
        r = step_dev()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    launches = 0
    binfos = []
    barrier(ws)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush()
            ev[i][0].record(stream)
            st_b, _, infos, ast, bi = step_dev()
            ev[i][1].record(stream)
            launches += bi.gpu_launches
            binfos.append(bi)
    torch.cuda.synchronize()
    barrier(ws)
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = allmax(sum(step_ms), ws)
    ms_per_step = total_ms / args.steps
    value = C5_ATLASES * args.steps / (total_ms / 1000.0)
    ok = int(sum(1 for s in ast if s == 0))
    stretch_b = float(np.mean([i.l2_stretch for i in infos if i.scale_index > 0]))

    # ---- e2e: host pointers from pinned memory (H2D + D2H inside the timed region)
    xy_p = torch.from_numpy(xy).pin_memory()
    cst_p = torch.from_numpy(cst).pin_memory()
    out_p = torch.empty(N * 32, dtype=torch.uint8).pin_memory()
    xy_h, cst_h = xy_p.numpy(), cst_p.numpy()
    from paper_2602_07782_b200 import PLACEMENT_DTYPE
    out_h = out_p.numpy().view(PLACEMENT_DTYPE)

    def step_host():
        return ctx.pack_many(xy_h, cst_h, abase, spec, res_xy=res, out=out_h,
                             stream=stream.cuda_stream)

    for _ in range(2):
        step_host()
    torch.cuda.synchronize()
    e2e_steps = max(5, args.steps // 2)
    e2e_ev, wall = [], []
    barrier(ws)
    for i in range(e2e_steps):
        flush()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        a.record(stream)
        step_host()
        b.record(stream)
        wall.append(time.perf_counter() - t0)
        e2e_ev.append((a, b))
    torch.cuda.synchronize()
    e2e_ms = allmax(sum(x.elapsed_time(y) for x, y in e2e_ev), ws) / e2e_steps
    wall_s = allmax(sum(wall), ws) / e2e_steps
    assert out_h.tobytes() == out_d.cpu().numpy().tobytes(), "host / device batch results differ"
    h2d = int(xy.nbytes + cst.nbytes + 4 * (4 * A + 1))
    d2h = int(N * 32 + A * (8 + 600))

    # ---- per-stage times of the batch (TABI_TIMING events, separate untimed steps)
    os.environ["TABI_TIMING"] = "1"
    stage = np.zeros(4)
    for _ in range(3):
        flush()
        stage += np.array(step_dev()[4].stage_ms[:4])
    stage /= 3
    os.environ["TABI_TIMING"] = "0"
    bi = binfos[-1]
    pk, pk_kind = peaks()
    sm_mhz = pk.get("sm_max_mhz", 1965.0)
    alu_peak = 148 * 128 * sm_mhz * 1e6 / 1e9  # G int32 lane-ops/s
    work = bi.work_pack + bi.work_profile
    stage_names = ["copies+reset", "proxies", "sort+slots", "pack_kernel (raster+pairs+Alg.4)"]
    kdom = int(np.argmax(stage))
    roof = {"kernel": ["reset", "proxy_kernel", "many_sort_prep_kernel", "many_kernel"][kdom],
            "bound": "alu", "unit": "Gop/s", "peak": alu_peak,
            "peak_kind": f"derived from {pk_kind} sm_max_mhz (148 SMs x 128 int32 lanes)",
            "stage_ms": {stage_names[i]: round(float(stage[i]), 4) for i in range(4)},
            "work_unit": "frontline column visits + footprint entries (batch kernel)",
            "work_per_launch": work, "traffic": None}
    if kdom == 3 and stage[3] > 0:
        roof["achieved"] = work / (stage[3] * 1e-3) / 1e9
        roof["frac"] = roof["achieved"] / alu_peak
    else:
        roof["achieved"] = roof["frac"] = None
    tr = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tr):
        roof["traffic"] = json.load(open(tr)).get("C5", {}).get("many_kernel")
    hbm_bytes = h2d + d2h
    line = {"metric": METRIC, "value": value, "unit": "atlases/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic (chartgen SplitMix64; configs[4] atlas i: seed 1000+i)",
            "config": {"workload": (f"C5 configs[4]: batch of {C5_ATLASES} tss atlases (200-2000 "
                                    "charts each, rho~U[0.3,1.5]) into 2048x2048, k=10, M=64, g=1, "
                                    f"LPT-sharded over {ws} GPU(s); one tabi_pack_many per rank "
                                    "per step"),
                       "latency_workload": (f"C3 configs[2]: 1572 tss charts into 4096x4096, "
                                            f"rho={C3_HEADLINE_RHO} (stretch ~1.39, the paper's "
                                            "2K TSS regime 1.38, P:796), k=10, t_opt=0, seeds 0-7"),
                       "l2": {"write": "flushed between steps (256 MB write, untimed)",
                              "write+read": "flushed between steps (256 MB write + 256 MB read)",
                              "none": "NOT flushed (warm-cache diagnostic, not a bench value)"
                              }[args.flush],
                       "parallelism": f"{C5_ATLASES} atlases per step sharded over {ws} GPU(s)"},
            "batch": {"atlases": C5_ATLASES, "atlases_this_rank": A, "charts_this_rank": N,
                      "device_atlases_per_s": value,
                      "e2e_atlases_per_s": C5_ATLASES * 1000.0 / e2e_ms,
                      "wall_atlases_per_s": C5_ATLASES / wall_s,
                      "ok_atlases_this_rank": ok, "l2_stretch_mean": stretch_b,
                      "candidates_evaluated": bi.candidates_evaluated,
                      "solo_atlases": bi.solo_atlases, "library_device_ms": bi.device_ms,
                      "per_gpu_busy_ms": sum(step_ms) / args.steps,
                      # batch-kernel load balance: last CTA's end after the
                      # median CTA's last item; mean CTA busy fraction
                      "kernel_tail_ms": bi.tail_ms, "kernel_busy_frac": bi.busy_frac,
                      "ranks_in_flight": bi.ranks_in_flight},
            "roofline": roof,
            "hbm_compulsory": {"bytes_per_step": hbm_bytes,
                               "gbs": hbm_bytes / (ms_per_step * 1e-3) / 1e9,
                               "frac_of_measured": hbm_bytes / (ms_per_step * 1e-3) / 1e9 /
                               pk.get("hbm_gbs", 6650.0)},
            "e2e": {"value": C5_ATLASES * 1000.0 / e2e_ms, "unit": "atlases/s",
                    "ms_per_step": e2e_ms, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "paper_context": PAPER_CONTEXT}
    line["p50_ms"] = line["p99_ms"] = line["l2_stretch"] = None
    if ws == 1 and not args.quick:
        c3 = {}
        for rho in (C3_HEADLINE_RHO, 0.5, 2.0):
            c3[f"rho_{rho}"] = c3_latency(ctx, stream, dev, rho, range(8), 25, flush)
        h = c3[f"rho_{C3_HEADLINE_RHO}"]
        line["p50_ms"], line["p99_ms"], line["l2_stretch"] = h["p50_ms"], h["p99_ms"], h["l2_stretch_mean"]
        line["c3"] = c3
        line["interactive_budget_ms"] = 15.0
        line["knob_sweep"] = knob_sweep(ctx, stream, dev, flush)
        line["shard_shares"] = shard_shares(ctx, stream, dev, flush, spec)
        # per-row cost of the headline pack vs the building-block floor
        cs, _ = workload("C3", 0, C3_HEADLINE_RHO)
        os.environ["TABI_TIMING"] = "1"
        xy1 = torch.from_numpy(cs.xy).to(dev)
        st1 = torch.from_numpy(cs.start).to(dev)
        fused = []
        for _ in range(5):
            flush()
            inf1 = ctx.pack(xy1, st1, spec_of(cs), stream=stream.cuda_stream)[2]
            fused.append(inf1.stage_ms[5])
        os.environ["TABI_TIMING"] = "0"
        fl = latency_floor(local)
        phases = 25  # barrier-separated steps per row
        line["latency_floor"] = dict(fl, phases_per_row=phases,
                                     row_floor_us=phases * fl["barrier_smem_exchange_ns"] / 2 / 1e3,
                                     fused_kernel_ms=statistics.median(fused), rows=inf1.rows,
                                     row_us_measured=statistics.median(fused) * 1e3 / max(1, inf1.rows))
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        rate, rate1, cores, n_done, wall_o = oracle_batch_rate(sets[::8])
        line["cpu_baseline"] = {"value": rate, "unit": "atlases/s", "cores": cores,
                                "kind": "oracle", "one_core_atlases_per_s": rate1,
                                "cpu_model": cpu_model(),
                                "sample": (f"{n_done} whole C5 atlases (every 8th of the batch, "
                                           f"rotating) in {wall_o:.1f} s, one oracle process per "
                                           f"core ({cores})")}
    if rank == 0:
        print(json.dumps(line))
    ctx.close()
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def run_single(args, ws, rank, local):
    """Round-1 single-pack bench (--workload C3 | C2 | C4 | C4P | C4X): one atlas per
    rank per step (weak scaling); kept for diagnostics and per-workload profiles."""
    import numpy as np
    import torch

    from paper_2602_07782_b200 import Context, spec_of
    from paper_2602_07782_b200 import build as nbuild
    if nbuild.needs_build():
        nbuild.build()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cs, desc = workload(args.workload, rank, args.rho)
    spec = spec_of(cs, **WORKLOAD_SPEC.get(args.workload, {}))
    ctx = Context(local, max_charts=max(cs.n_charts, 1024), max_vertices=cs.n_vertices + 16,
                  max_atlas_side=max(cs.atlas_w, cs.atlas_h))
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    xy_d, st_d = torch.from_numpy(cs.xy).to(dev), torch.from_numpy(cs.start).to(dev)
    out_d = torch.empty(cs.n_charts * 32, dtype=torch.uint8, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    os.environ["TABI_TIMING"] = "0"
    for _ in range(args.warmup):
        ctx.pack(xy_d, st_d, spec, out=out_d, stream=stream.cuda_stream)
    torch.cuda.synchronize()
    span, launches, info = [], 0, None
    barrier(ws)
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            if args.flush != "none":
                flush.zero_()
            info = ctx.pack(xy_d, st_d, spec, out=out_d, stream=stream.cuda_stream)[2]
            span.append(info.device_ms)
            launches += info.gpu_launches
    torch.cuda.synchronize()
    total = allmax(sum(span), ws)
    os.environ["TABI_TIMING"] = "1"
    stage = np.zeros(8)
    for _ in range(min(args.steps, 10)):
        flush.zero_()
        stage += np.array(ctx.pack(xy_d, st_d, spec, out=out_d, stream=stream.cuda_stream)[2].stage_ms[:8])
    stage /= min(args.steps, 10)
    os.environ["TABI_TIMING"] = "0"
    e2e = []
    for _ in range(10):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        ctx.pack(cs.xy, cs.start, spec, stream=stream.cuda_stream)
        b.record(stream)
        e2e.append((a, b))
    torch.cuda.synchronize()
    e2e_ms = allmax(sum(x.elapsed_time(y) for x, y in e2e), ws) / 10
    names = ["h2d", "proxies", "sort", "profiles", "offsets_locks", "fold_push", "select", "d2h"]
    span.sort()
    line = {"metric": METRIC, "value": ws * args.steps / (total / 1000.0), "unit": "atlases/s",
            "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "int32", "data": "synthetic (chartgen, seed = rank)",
            "config": {"workload": desc, "parallelism": f"{ws} independent packs per step"},
            "p50_ms": statistics.median(span), "p99_ms": span[int(0.99 * (len(span) - 1))],
            "l2_stretch": info.l2_stretch, "scale_index": info.scale_index, "rows": info.rows,
            "prefix_rows": info.prefix_rows,
            "stage_ms": {names[i]: round(float(stage[i]), 5) for i in range(8)},
            "e2e": {"value": ws * 1000.0 / e2e_ms, "unit": "atlases/s", "ms_per_step": e2e_ms,
                    "h2d_bytes_per_step": int(cs.xy.nbytes + cs.start.nbytes),
                    "d2h_bytes_per_step": int(cs.n_charts * 32)},
            "gpu_launches": launches, "clocks": clk.summary()}
    if rank == 0:
        print(json.dumps(line))
    ctx.close()


if __name__ == "__main__":
    main()
