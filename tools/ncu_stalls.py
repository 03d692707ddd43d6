"""Top stall reasons per source line of one kernel (ncu source page).
usage: python tools/ncu_stalls.py REPORT KERNEL_REGEX FUNC_SUBSTR [TOP]"""
import csv, io, subprocess, sys
rep, kern, fsel = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name", "regex:" + kern], capture_output=True, text=True).stdout
agg, fname, func, cols = {}, "?", "?", None
for row in csv.reader(io.StringIO(out)):
    if not row: continue
    if row[0] == "File Path": fname = row[1].split("/")[-1]; continue
    if row[0] == "Function Name": func = row[1]; continue
    if row[0] == "Line No": cols = row; continue
    if fsel not in func or not row[0].isdigit() or cols is None: continue
    st = {c: float(row[i] or 0) for i, c in enumerate(cols) if c.startswith("stall_") and "Not Issued" not in c and row[i] not in ("", "-")}
    a = agg.setdefault((fname, int(row[0])), [0.0, {}, row[1].strip()[:70]])
    for k, v in st.items():
        a[1][k] = a[1].get(k, 0) + v
        a[0] += v
tot = sum(v[0] for v in agg.values()) or 1
allr = {}
for v in agg.values():
    for k, x in v[1].items(): allr[k] = allr.get(k, 0) + x
print("all:", ", ".join("%s %.1f%%" % (k[6:], 100 * x / tot) for k, x in sorted(allr.items(), key=lambda kv: -kv[1])[:8]))
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    rs = sorted(v[1].items(), key=lambda kv: -kv[1])[:3]
    print("%-16s %5d %5.1f%%  %s  | %s" % (k[0], k[1], 100 * v[0] / tot, ", ".join("%s %.0f%%" % (r[6:], 100 * x / max(v[0], 1)) for r, x in rs), v[2]))
