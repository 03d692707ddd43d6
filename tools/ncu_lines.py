"""Aggregate an ncu source page per CUDA source line: warp-stall samples and warp instructions.

usage: python tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX [TOP]
(reads `ncu -i REPORT --page source --csv --print-source cuda,sass`; the CUDA-line rows carry the
per-line totals in columns 4 (stall samples) and 7 (instructions executed))."""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name", "regex:" + kern], capture_output=True, text=True).stdout
agg = {}
fname = "?"
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if not row[0].isdigit() or len(row) < 8:
        continue
    try:
        samples, inst = float(row[4] or 0), float(row[7] or 0)
    except ValueError:
        continue
    a = agg.setdefault((fname, int(row[0])), [0.0, 0.0, row[1].strip()[:100]])
    a[0] += samples
    a[1] += inst
tot_s = sum(v[0] for v in agg.values()) or 1.0
tot_i = sum(v[1] for v in agg.values()) or 1.0
print("total stall samples %.0f, warp instructions %.4g" % (tot_s, tot_i))
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print("%-14s %5d  stall %5.1f%%  inst %5.1f%%  %s" % (k[0], k[1], 100 * v[0] / tot_s, 100 * v[1] / tot_i, v[2]))
