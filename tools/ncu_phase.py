"""Warp/thread instructions and stall samples of one kernel in an ncu report, grouped by source-line ranges.
usage: python tools/ncu_phase.py REPORT KERNEL_REGEX FUNC_SUBSTR '{"name": ("file", lo, hi), ...}'"""
import csv, io, subprocess, sys
rep, kern, fsel = sys.argv[1], sys.argv[2], sys.argv[3]
ranges = eval(sys.argv[4])   # {"name": ("file", lo, hi), ...}
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "--kernel-name", "regex:" + kern], capture_output=True, text=True).stdout
fname = func = "?"; cols = None; agg = {}
for row in csv.reader(io.StringIO(out)):
    if not row: continue
    if row[0] == "File Path": fname = row[1].split("/")[-1]; continue
    if row[0] == "Function Name": func = row[1]; continue
    if row[0] == "Line No": cols = row; continue
    if fsel not in func or not row[0].isdigit() or cols is None: continue
    try:
        ln = int(row[0]); wv = row[cols.index("Instructions Executed")]; tv = row[cols.index("Thread Instructions Executed")]; wi = float(wv) if wv not in ("","-") else 0.0; ti = float(tv) if tv not in ("","-") else 0.0
        sv = row[cols.index("Warp Stall Sampling (All Samples)")]; st = float(sv) if sv not in ("", "-") else 0.0
    except (ValueError, IndexError):
        continue
    key = "other"
    for k, (f, a, b) in ranges.items():
        if f in fname and a <= ln <= b: key = k
    v = agg.setdefault(key, [0, 0, 0]); v[0] += wi; v[1] += ti; v[2] += st
T = [sum(v[i] for v in agg.values()) for i in range(3)]
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print("%-12s warp %6.1f%% (%.3g)  thr/inst %5.1f  stall %5.1f%%" % (k, 100*v[0]/T[0], v[0], v[1]/max(v[0],1), 100*v[2]/T[2]))
