"""Update profiles/traffic.json from one `ncu --set full` report of the raster kernels.

For each kernel: DRAM bytes (read + write) per launch -> bench.py's roofline.traffic / roofline.hbm, and
the warp efficiency (active lanes per executed warp instruction / 32) of the whole kernel and of its
coverage-test loop (the source lines of vis_mask_fast / vis_mask in k_raster.cu) -> roofline.warp_efficiency.

usage: python tools/update_traffic.py REPORT.ncu-rep CONFIG [kernel_regex=name ...]
e.g.   python tools/update_traffic.py gpurun_out/prof_c4.ncu-rep C4 'k4l_raster_fwd<0>=k4l_raster_fwd' \
           'k6v_raster_bwd=k6v_raster_bwd'
"""
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "": 1.0}


def raw_rows(rep):
    """Rows of the raw page with every value converted to base units (bytes for byte metrics)."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for h, u, v in zip(hdr, units, r):
            if u in SCALE and u:
                try:
                    v = float(v) * SCALE[u]
                except ValueError:
                    pass
            d[h] = v
        res.append(d)
    return res


def coverage_loop_efficiency(rep, func_sub):
    """threads / warp instruction over the source lines of the coverage loops (k_raster.cu): k4l_raster_fwd's
    lines between its `coverage loop: begin` / `end` markers, else vis_mask_fast / vis_mask."""
    src = open(os.path.join(ROOT, "paper_2602_07860_b200", "csrc", "k_raster.cu")).read().split("\n")
    lines = set()
    if func_sub.startswith("k4l"):
        b = next(i for i, l in enumerate(src) if "coverage loop: begin" in l)
        e = next(i for i in range(b, len(src)) if "coverage loop: end" in src[i])
        lines.update(range(b + 1, e + 2))
    else:
        for name in ("vis_mask_fast", "vis_mask"):
            start = next(i for i, l in enumerate(src) if re.match(r"__device__ __forceinline__ (bool|void) %s\(" % name, l))
            end = next(i for i in range(start + 1, len(src)) if src[i].startswith("}"))
            lines.update(range(start + 1, end + 2))
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    fname = func = None
    cols = None
    wi = ti = 0.0
    for row in csv.reader(io.StringIO(out)):
        if not row:
            continue
        if row[0] == "File Path":
            fname = row[1]
            continue
        if row[0] == "Function Name":
            func = row[1]
            continue
        if row[0] == "Line No":
            cols = row
            continue
        if not (fname and fname.endswith("k_raster.cu") and func and func_sub in func and row[0].isdigit()):
            continue
        try:
            ln = int(row[0])
            w = float(row[cols.index("Instructions Executed")] or 0)
            t = float(row[cols.index("Thread Instructions Executed")] or 0)
        except (ValueError, IndexError):
            continue
        if ln in lines:
            wi += w
            ti += t
    return ti / wi / 32.0 if wi > 0 else None


def main():
    rep, cfg = sys.argv[1], sys.argv[2]
    pairs = [a.split("=", 1) for a in sys.argv[3:]]
    path = os.path.join(ROOT, "profiles", "traffic.json")
    data = json.load(open(path)) if os.path.exists(path) else {}
    ent = data.setdefault(cfg, {})
    weff = ent.setdefault("warp_efficiency", {})
    rows = raw_rows(rep)
    for pat, name in pairs:
        hits = [r for r in rows if pat in r.get("Kernel Name", "")]
        if not hits:
            print("no kernel matching", pat)
            continue
        r = hits[-1]
        rd = float(r["dram__bytes_read.sum"])
        wr = float(r["dram__bytes_write.sum"])
        ent[name] = rd + wr
        ratio = float(r["smsp__thread_inst_executed_per_inst_executed.ratio"]) / 32.0
        loop = coverage_loop_efficiency(rep, pat.split("<")[0])
        weff[name] = {"kernel": ratio, "coverage_loop": loop}
        print(name, "dram", rd + wr, "warp eff", ratio, "coverage loop", loop)
    data["_note"] = ("per config and kernel: DRAM bytes (read + write) per launch and the warp efficiency "
                     "(active lanes per executed warp instruction / 32; whole kernel and coverage-test loop) "
                     "from one ncu --set full capture (tools/update_traffic.py); bench.py reports them in "
                     "roofline.traffic / roofline.hbm / roofline.warp_efficiency")
    json.dump(data, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
