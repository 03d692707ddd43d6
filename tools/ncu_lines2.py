"""Per-source-line warp instructions, thread instructions and stall samples of one kernel in an ncu report.

usage: python tools/ncu_lines2.py REPORT.ncu-rep KERNEL_REGEX [TOP] [FUNC_SUBSTR]
FUNC_SUBSTR picks one instantiation when the regex matches several (e.g. '(bool)0')."""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
fsel = sys.argv[4] if len(sys.argv) > 4 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name", "regex:" + kern], capture_output=True, text=True).stdout
agg, fname, func, cols = {}, "?", "?", None
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row[0] == "Function Name":
        func = row[1]
        continue
    if row[0] == "Line No":
        cols = row
        continue
    if fsel and fsel not in func:
        continue
    if not row[0].isdigit() or cols is None:
        continue
    try:
        s = float(row[cols.index("Warp Stall Sampling (All Samples)")] or 0)
        wi = float(row[cols.index("Instructions Executed")] or 0)
        ti = float(row[cols.index("Thread Instructions Executed")] or 0)
    except (ValueError, IndexError):
        continue
    a = agg.setdefault((fname, int(row[0])), [0.0, 0.0, 0.0, row[1].strip()[:90]])
    a[0] += s; a[1] += wi; a[2] += ti
T = [sum(v[i] for v in agg.values()) or 1.0 for i in range(3)]
print("stall samples %.4g  warp inst %.4g  thread inst %.4g  (%.1f threads/inst)" % (T[0], T[1], T[2], T[2] / T[1]))
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][2])[:top]:
    print("%-18s %5d  thr %5.1f%%  warp %5.1f%%  (%4.1f/inst)  stall %5.1f%%  %s" % (
        k[0], k[1], 100 * v[2] / T[2], 100 * v[1] / T[1], v[2] / max(v[1], 1), 100 * v[0] / T[0], v[3]))
