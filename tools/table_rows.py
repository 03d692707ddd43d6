"""Markdown rows of BASELINE.md section 3 from bench.py JSON lines (tools/baseline_table.sh)."""
import json
import sys


def fmt(x, f="%.3g"):
    return "-" if x is None else f % x


print("| Config | GPUs | blurred images/s (fwd+bwd) | e2e images/s | ms/step | barycentric evals/s (executed / necessary) "
      "| % FP32 peak (kernel) | % HBM peak | warp eff. (kernel lanes active / coverage-test lanes useful) | CPU oracle images/s (cores) |")
print("|---|---|---|---|---|---|---|---|---|---|")
for path in sys.argv[1:]:
    try:
        d = json.loads(open(path).read().strip().splitlines()[-1])
    except Exception as e:   # noqa: BLE001
        print("| %s | failed: %s |" % (path, e))
        continue
    r, c = d["roofline"], d["config"]
    ev = d.get("barycentric_evals_per_s", {})
    we = r.get("warp_efficiency") or {}
    cb = d.get("cpu_baseline") or {}
    e2e = (d.get("e2e") or {}).get("value")
    name = "%s %d x %d^2, %d F, N=%d%s" % (c["workload"], c["images"], c["H"], c["faces"], c["subframes"],
                                           " (CUDA graph)" if c.get("cuda_graph") else "")
    print("| %s | %d | %s | %s | %s | %s / %s | %s (%s) | %s | %s / %s | %s (%s) |" % (
        name, d["n_gpus"], fmt(d["value"], "%.1f"), fmt(e2e, "%.1f"), fmt(d["ms_per_step"], "%.3f"),
        fmt(ev.get("executed")), fmt(ev.get("necessary")), fmt(100 * r["frac"], "%.2f"), r["kernel"],
        fmt(None if r.get("hbm_frac") is None else 100 * r["hbm_frac"], "%.2f"), fmt(we.get("kernel"), "%.2f"),
        fmt(we.get("coverage_loop_useful_lanes"), "%.3f"), fmt(cb.get("value"), "%.3g"), cb.get("cores", "-")))
