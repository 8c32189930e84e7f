"""Summarise an ncu report (run here, no GPU needed):

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--json out.json]

Prints, per captured kernel: duration, SM/memory throughput, occupancy,
registers, IPC, active threads per warp (durations in ns, bytes in bytes,
converted from the report's units), DRAM bytes (read+write -> the
`traffic` of bench.py's roofline) and the top warp-stall reasons.
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem_throughput_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "launch__registers_per_thread": "registers",
    "sm__inst_executed.avg.per_cycle_active": "ipc_active",
    "smsp__thread_inst_executed_per_inst_executed.ratio": "active_threads_per_warp",
    "smsp__inst_executed.sum": "warp_instructions",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wavefronts",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
}


def main():
    rep = sys.argv[1]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    unit_of = dict(zip(hdr, units))
    scale = {"nsecond": 1.0, "ns": 1.0, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6,
             "second": 1e9, "s": 1e9,
             "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    out = []
    for r in data:
        d = dict(zip(hdr, r))
        name = d.get("Kernel Name", "?").split("(")[0].split("::")[-1]
        rec = {"kernel": name}
        for k, v in KEYS.items():
            if k in d:
                try:
                    rec[v] = float(d[k].replace(",", "")) * scale.get(unit_of.get(k, ""), 1.0)
                except ValueError:
                    rec[v] = d[k]
        stalls = {}
        for k, v in d.items():
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    stalls[k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = float(v)
                except ValueError:
                    pass
        rec["top_stalls"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:5])
        if "dram_read_bytes" in rec and "dram_write_bytes" in rec:
            rec["dram_bytes"] = rec["dram_read_bytes"] + rec["dram_write_bytes"]
        out.append(rec)
    for rec in out:
        print(json.dumps(rec))
    if "--json" in sys.argv:
        json.dump(out, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)


if __name__ == "__main__":
    main()
