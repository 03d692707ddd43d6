"""Markdown tables from an ncu launch list (--metrics gpu__time_duration.sum --csv) and an ncu --set full
report: per-kernel launch shares, and the headline counters of the profiled kernels.

usage: python tools/summarize_profiles.py LAUNCHES.csv REPORT.ncu-rep"""
import csv
import io
import subprocess
import sys
from collections import OrderedDict


def launches(path):
    rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
    hdr = rows[0]
    ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = OrderedDict()
    unit = None
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        unit = r[ui]
        v = float(r[vi].replace(",", ""))
        name = r[ki].split("(")[0]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}.get(unit, 1e-6)
    tot = sum(v[1] for v in agg.values())
    out = ["| kernel | launches | total ms | ms / launch | share |", "|---|---|---|---|---|"]
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append("| `%s` | %d | %.3f | %.3f | %.1f%% |" % (k[:70], n, t * scale, t * scale / n, 100 * t / tot))
    return "\n".join(out)


METRICS = [
    ("duration (ms)", "gpu__time_duration.sum", 1e-6),
    ("registers / thread", "launch__registers_per_thread", 1),
    ("CTAs / SM limit (regs, smem)", None, None),
    ("warps active (% of peak)", "sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    ("issue active (% of peak)", "smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    ("thread inst / warp inst", "smsp__thread_inst_executed_per_inst_executed.ratio", 1),
    ("smem bank conflicts", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", 1),
    ("DRAM read (MB)", "dram__bytes_read.sum", 1e-6),
    ("DRAM write (MB)", "dram__bytes_write.sum", 1e-6),
    ("warp instructions", "smsp__inst_executed.sum", 1),
    ("SM active / elapsed cycles", "ACTIVE_FRAC", 1),
]


def full(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    kern = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        kern.append((d["Kernel Name"].split("(")[0], d, u))
    lines = ["| metric | " + " | ".join("`%s`" % k[0].split("::")[-1] for k in kern) + " |",
             "|---|" + "---|" * len(kern)]
    for label, m, sc in METRICS:
        if m is None:
            vals = ["%s, %s" % (d.get("launch__occupancy_limit_registers", "?"), d.get("launch__occupancy_limit_shared_mem", "?"))
                    for _, d, _ in kern]
        elif m == "ACTIVE_FRAC":   # launch tail: SMs without a resident warp
            vals = []
            for _, d, _ in kern:
                try:
                    vals.append("%.3f" % (float(d["sm__cycles_active.avg"].replace(",", "")) /
                                          float(d["sm__cycles_elapsed.avg"].replace(",", ""))))
                except (KeyError, ValueError):
                    vals.append("-")
        else:
            vals = []
            for _, d, u in kern:
                v = d.get(m)
                if v is None:
                    vals.append("-")
                    continue
                x = float(v.replace(",", ""))
                un = u.get(m, "")
                if m == "gpu__time_duration.sum":
                    x *= {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1, "msecond": 1}.get(un, 1e-6)
                    vals.append("%.3f" % x)
                elif m.startswith("dram__bytes"):
                    x *= {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1, "Gbyte": 1e3}.get(un, 1e-6)
                    vals.append("%.1f" % x)
                else:
                    vals.append("%.4g" % x)
        lines.append("| %s | %s |" % (label, " | ".join(vals)))
    return "\n".join(lines)


if __name__ == "__main__":
    print(launches(sys.argv[1]))
    print()
    print(full(sys.argv[2]))
