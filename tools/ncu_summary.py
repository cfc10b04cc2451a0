#!/usr/bin/env python
"""Summarise ncu artefacts into text committed under profiles/.

  ncu_summary.py launches <launches.csv>            per-kernel share of a launch list
  ncu_summary.py report <x.ncu-rep> <evals/launch>  key counters of a --set full capture
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_sector_hit_rate.pct",
        "lts__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sectors.sum.per_second", "dram__bytes.sum.per_second",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum"]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "")[:48]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += float(r[vi].replace(",", ""))
    tot = sum(a[1] for a in agg.values())
    out = [f"{'kernel':48s} {'launches':>8s} {'total_us':>10s} {'avg_us':>9s} {'share':>6s}"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{k:48s} {n:8d} {t / 1e3:10.1f} {t / n / 1e3:9.2f} {100 * t / tot:5.1f}%")
    return "\n".join(out)


def report(path, evals=None):
    raw = subprocess.check_output(["ncu", "-i", path, "--page", "raw", "--csv"], stderr=subprocess.DEVNULL).decode()
    r = list(csv.reader(io.StringIO(raw)))
    h, units = r[0], r[1]
    out = []
    for row in r[2:]:
        name = row[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        out.append(f"kernel: {name[:100]}")
        vals = {}

        def num(k):
            return float(vals.get(k, "0").replace(",", ""))
        for k in KEYS:
            if k in h:
                i = h.index(k)
                vals[k] = row[i]
                out.append(f"  {k:72s} {row[i]:>16s} {units[i]}")
        if evals:
            dram = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
            unit = units[h.index("dram__bytes_read.sum")]
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
            out.append(f"  evals/launch {evals:.0f}: DRAM bytes/eval {dram * scale / evals:.4f}; "
                       f"global ld wavefronts/eval {num('l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum') / evals:.3f}; "
                       f"shared wavefronts/eval {num('l1tex__data_pipe_lsu_wavefronts_mem_shared.sum') / evals:.3f}; "
                       f"sectors/request {num('l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum') / max(1, num('l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum')):.2f}; "
                       f"warp instr/warp-eval {num("smsp__inst_executed.sum") / (evals / 32):.1f}")
        if "lts__t_sectors.sum.per_second" in vals:
            u = units[h.index("lts__t_sectors.sum.per_second")]
            per = {"sector/ns": 1e9, "sector/us": 1e6, "sector/ms": 1e3, "sector/s": 1.0}.get(u, 1.0)
            sec_s = float(vals["lts__t_sectors.sum.per_second"].replace(",", "")) * per
            out.append(f"  achieved L2 throughput {sec_s * 32 / 1e9:.0f} GB/s (32-byte sectors; "
                       f"{num('lts__throughput.avg.pct_of_peak_sustained_elapsed'):.1f}% of the L2 peak)")
    return "\n".join(out)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        print(launches(sys.argv[2]))
    else:
        print(report(sys.argv[2], float(sys.argv[3]) if len(sys.argv) > 3 else None))
