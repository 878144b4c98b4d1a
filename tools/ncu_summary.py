"""Summarise an `ncu --set full` capture of one kernel launch into profiles/.

    python tools/ncu_summary.py gpurun_out/r01/k_engine_C2.ncu-rep profiles/r01_k_engine_C2 \
        [--workload C2] [--algorithmic-bytes B]

Writes <out>.txt (the key counters, readable).
"""
import argparse
import csv
import io
import json
import subprocess
from pathlib import Path

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "L1 global load sectors"),
    ("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "L1 global load requests"),
    ("l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum", "local (spill) load sectors"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "instructions"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
]
STALLS = ["long_scoreboard", "barrier", "wait", "short_scoreboard", "branch_resolving", "selected",
          "no_instructions", "not_selected", "lg_throttle", "math_pipe_throttle", "membar", "mio_throttle"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return [dict(zip(rows[0], zip(rows[1], r))) for r in rows[2:]]


def num(v):
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return None


def to_bytes(val, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    return val * scale.get(unit, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("out")
    ap.add_argument("--workload", default="C2")
    ap.add_argument("--algorithmic-bytes", type=float, default=None)
    a = ap.parse_args()
    launches = raw(a.rep)
    lines = [f"ncu --set full capture: {a.rep}", ""]
    summary = {}
    for i, d in enumerate(launches):
        name = d.get("Kernel Name", ("", "?"))[1]
        lines.append(f"launch {i}: {name[:100]}")
        for k, label in KEYS:
            if k in d:
                u, v = d[k]
                lines.append(f"  {label:34s} {v} {u}")
        rd = d.get("dram__bytes_read.sum")
        wr = d.get("dram__bytes_write.sum")
        if rd and wr:
            tb = to_bytes(num(rd[1]), rd[0]) + to_bytes(num(wr[1]), wr[0])
            dur = d.get("gpu__time_duration.sum")
            ms = num(dur[1]) * {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3,
                                "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3}[dur[0]]
            lines.append(f"  {'DRAM bytes per launch':34s} {tb / 1e9:.3f} GB -> {tb / ms / 1e6:.1f} GB/s")
            if a.algorithmic_bytes:
                lines.append(f"  {'algorithmic bytes (bench.py)':34s} {a.algorithmic_bytes / 1e9:.3f} GB "
                             f"(traffic / algorithmic = {tb / a.algorithmic_bytes:.2f})")
            summary = {"dram_bytes": tb, "ms": ms}
        sec = d.get("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum")
        req = d.get("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum")
        if sec and req and num(req[1]):
            lines.append(f"  {'global load sectors per request':34s} {num(sec[1]) / num(req[1]):.2f}")
        tot = sum(num(d.get(f"smsp__pcsamp_warps_issue_stalled_{s}", ("", "0"))[1]) or 0 for s in STALLS)
        if tot:
            lines.append("  warp-stall samples:")
            for s in sorted(STALLS, key=lambda s: -(num(d.get(f"smsp__pcsamp_warps_issue_stalled_{s}", ("", "0"))[1]) or 0)):
                x = num(d.get(f"smsp__pcsamp_warps_issue_stalled_{s}", ("", "0"))[1]) or 0
                if x:
                    lines.append(f"    {s:22s} {100 * x / tot:5.1f}%")
    Path(a.out + ".txt").write_text("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
