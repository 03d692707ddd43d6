"""Write profiles/r2e_summary.md (round 2, fifth session) from the gpurun artefacts in gpurun_out/:
tools/baseline_table.sh (table_*.json: one bench line per config), tools/profile_tag.sh (TAG=r2e) (r2e_launches_C4.csv,
the ncu launch list of the default bench; prof_r2e_c4.ncu-rep, ncu --set full of K4 and K6 on C4).
Copies the raw launch list and the ncu details page into profiles/ as r2e_*.

usage: python tools/write_summary_r2e.py   (from the repo root)"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
sys.path.insert(0, os.path.join(ROOT, "tools"))
import summarize_profiles as sp  # noqa: E402


def load(name):
    p = os.path.join(OUT, name + ".json")
    if not os.path.exists(p):
        return None
    return json.loads(open(p).read().strip().splitlines()[-1])


def sh(cmd):
    return subprocess.run(cmd, capture_output=True, text=True).stdout


HISTORY = """| change (round 2) | fwd ms | bwd ms | step ms | images/s |
|---|---|---|---|---|
| end of round 1 (visibility buffer of every sub-frame, 2 B per pixel) | 7.06 | 6.83 | 14.57 | 1098 |
| first session of round 2 (span raster tried; K6 fixed-point moments; bounded cache, NCCL step) | 7.07 | 6.92 | 14.65 | 1092 |
| K6 visibility gather (`k_gather.cu`): whole chunks as one group, thread per won pair | 7.07 | 3.67 | 11.40 | 1403 |
| K6 gather: super-groups of up to 16 sub-frames over several chunks, run-aggregated moments | 7.06 | 3.58 | 11.15 | 1436 |
| K4 lean (`k4l_raster_fwd`): per-footprint record lists, lane pixel in shared memory | 6.87 | 3.58 | 11.11 | 1440 |
| (tried) K4 warp-specialised producer/consumer (`BLURRAST_FWD=pipe`), 4 or 8 producer warps | 8.8-9.2 | - | - | - |
| (tried) K4 per-face depth cull of faces turned away; warp-queue / two-pass compacted staging; paired staging | 7.2-8.2 | - | - | - |
| K6 gather at 5 CTAs/SM (48 registers), slot words packed | 6.84 | 3.37 | 10.89 | 1469 |
| K4 list-level skip of the faces turned away from the camera (exact corner depth bound) | 6.14 | 3.37 | 10.18 | 1571 |
| fifth session: records evaluated about the moving vertex a(tau) (numerics; no time change) | 6.15 | 3.36 | 10.16 | 1574 |
| (tried) K4 order (i), pixel-major (`BLURRAST_FWD=pixmajor`, `r2c_order_i_vs_ii.md`) | 20.1-24.0 | - | - | - |
| K4 REDUX warp max for the list skip, `__frcp_rn`, branch-free footprint masks | 5.92 | 3.36 | 9.95 | 1608 |
| (tried) K4 super-groups of consecutive chunks (`BLURRAST_FWD=sg`); group caps 192/256/320 pairs | 6.13-6.68 | - | - | - |
| (tried) K4 next chunk's bin entries prefetched by `cp.async` (`BR_K4L_PREF`) | 6.03 | - | - | - |
| K6 run moments from per-row prefix sums (two lookups per run) | 5.92 | 2.90 | 9.50 | 1685 |
| visibility cache written / read evict-first (streaming) | 5.90 | 2.91 | 9.46 | 1691 |
| (tried) K4 lazy staging of the faces turned away (`BR_K4L_LAZY`) | 6.44 | - | - | - |
| soft: Cartesian closest points (C5 sliver parity fix; soft C4 +2%) | 5.90 | 2.91 | 9.42 | 1699 |
| K6 recompute path (no cache) with run-aggregated moments; backward record stage 256 -> 384 (C5 378.8 -> 375.1 ms) | 5.86 | 2.88 | 9.41 | 1701 |
| (tried) K4 record written before the footprint masks (`BR_STAGE_EARLY`); whole record per pair in one request (`BR_K4L_ONELOAD`) | 5.88-5.90 | - | - | - |
| (tried) K4 next chunk header / next taus one phase ahead (`BR_K4L_TPREF`); bin sizes of 32 chunks in one load (`BR_K4L_NWIN`) | 5.95-5.96 | - | - | - |
| K4 coverage loop keeps the winner's edge values; shading reads only (invD, face) (`BR_K4L_EKEEP`) | 5.75 | 2.88 | 9.28 | 1724 |
| K4 48-B stage records + separate (invD, face) pairs: conflict-free record stores (`BR_K4L_R48`) | 5.64 | 2.88 | 9.18 | 1743 |
| K4 per-warp counter clears, two barriers per group instead of three (`BR_K4L_WCLR`) | 5.51 | 2.88 | 9.06 | 1765 |
| (tried) K4 stage reads its taus from the global schedule (`BR_K4L_GTAU`) | 5.52 | - | - | - |
| (tried) K4 next chunk's header copied to shared memory by `cp.async` during the stage (`BR_K4L_HPREF`) | 5.98 | - | - | - |"""


def row(label, d):
    r = d["roofline"]
    km = r.get("kernels_ms")
    soft = "%.1f / %.1f" % (km["k8_soft_fwd"], km["k9_soft_bwd"]) if km else "-"
    e2e = "%.1f" % d["e2e"]["value"] if d.get("e2e") else "-"
    hb = "-" if r.get("hbm_frac") is None else "%.4f" % r["hbm_frac"]
    passes = d["config"].get("passes_per_rank", 1)
    return "| %s | %.1f | %.3f | %.3f | %.3f | %s | %s | %d | %s, %.4f | %s | %s MHz %s |" % (
        label, d["value"], d["ms_per_step"], r["fwd_raster_ms"], r["bwd_raster_ms"], soft, e2e, passes,
        r["kernel"], r["frac"], hb, d["clocks"]["sm_mhz"], d["clocks"]["reasons"])


def main():
    lines = [("C1 (`--config C1 --graph --steps 50`)", "table_C1"),
             ("C2 (`--config C2 --graph --steps 50`)", "table_C2"),
             ("C2 eager", "table_C2_eager"),
             ("C3 (`--config C3 --graph --steps 50`)", "r2e_bench_C3"),
             ("C3 eager", "table_C3_eager"),
             ("C4 (`python bench.py`, the default)", "r2e_bench_C4"),
             ("C4 soft coverage (`--delta 1e-4`)", "table_C4_soft"),
             ("C5 (`--config C5 --steps 3`)", "r2e_bench_C5"),
             ("C5 soft coverage (`--config C5 --delta 1e-4 --steps 1`)", "table_C5_soft")]
    rows_b = [row(lab, d) for lab, d in ((lab, load(n)) for lab, n in lines) if d is not None]
    c4 = load("r2e_bench_C4")
    ref = load("bench_ref")
    launches = os.path.join(OUT, "r2e_launches_C4.csv")
    rep = os.path.join(OUT, "prof_r2e_c4.ncu-rep")
    tab_l = sp.launches(launches)
    tab_f = sp.full(rep)
    subprocess.run(["cp", launches, os.path.join(PROF, "r2e_launches_C4.csv")])
    open(os.path.join(PROF, "r2e_ncu_details_raster_C4.csv"), "w").write(
        sh(["ncu", "-i", rep, "--page", "details", "--csv"]))
    k4s = sh([sys.executable, os.path.join(ROOT, "tools", "ncu_stalls.py"), rep, "k4l_raster_fwd", "k4l", "10"])
    k6s = sh([sys.executable, os.path.join(ROOT, "tools", "ncu_stalls.py"), rep, "k6v_raster_bwd", "k6v", "10"])
    rc = c4["roofline"]
    cb = c4["cpu_baseline"]
    we = rc.get("warp_efficiency") or {}
    refl = ""
    if ref is not None:
        refl = ("`--impl reference` (the fp64 oracle, %s host threads): %.2f images/s, %.0f ms per step "
                "(%s).\n" % (ref["cpu_baseline"]["cores"], ref["value"], ref["ms_per_step"], ref["cpu_baseline"]["sample"]))
    md = f"""# Round 2 (fifth session) profile summary (B200, sm_100a)

Generated by `tools/write_summary_r2e.py` from `tools/baseline_table.sh` (one bench line per config, one
gpurun call on one box) and `tools/profile_tag.sh (TAG=r2e)` (ncu launch list + `ncu --set full` of K4 = `k4l_raster_fwd`
and K6 = `k6v_raster_bwd` on C4).  Raw files: `r2e_launches_C4.csv` (ncu launch list), `r2e_ncu_details_raster_C4.csv`
(ncu details of K4 and K6), `traffic.json` (DRAM bytes per launch and warp efficiencies -> `roofline.traffic`,
`roofline.hbm`, `roofline.warp_efficiency`), `r2e_checked_build.log` (the checked build over the GPU tests, final code; `r2d_checked_build.log` the fourth session's, `r2c_checked_build.log` the third session's),
`r2c_order_i_vs_ii.md` (K4 evaluation orders), `r2c_variants_parity.log` (the A/B forwards over the parity tests), `r2e_gpu_tests.log` (this session's `pytest -m gpu` + smoke on the final code).  Earlier sessions: `r2d_summary.md` (the full C1-C5 table, before EKEEP / R48), `r2c_summary.md`, `r2b_summary.md`, `r2_summary.md`; round 1: `r1_summary.md`.

## Bench lines (1 B200)

| workload | images/s | ms/step | K4 fwd ms | K6 bwd ms | soft K8 / K9 ms | e2e images/s | passes | roofline kernel, frac (alu, derived 74.4 TF) | hbm_frac | clocks |
|---|---|---|---|---|---|---|---|---|---|---|
{chr(10).join(rows_b)}

The timed step is `dist.ShardedStep` on a 1-rank NCCL group (its gradient all-reduce runs).  C5 runs its
64 images in passes whose per-sub-frame winner index fits the 1 GiB visibility-cache budget (round 1
kept a 34 GB buffer for all of them: 116.5 images/s; round 2 with <= 1 GiB: {load('r2e_bench_C5')['value'] if load('r2e_bench_C5') else float('nan'):.1f}).

CPU oracle (fp64, binned, {cb['cores']} host threads): {cb['value']:.2f} images/s on C4 ({cb['sample']}).
{refl}Measured FFMA probe: {c4['ffma_measured_tflops']:.1f} TFLOP/s (derived peak 74.4).

C4 forward census per launch: {rc['executed_pair_tests_per_launch']:.3e} executed (pixel, face, sub-frame) tests,
{rc['necessary_pairs_per_launch']:.3e} covered pairs, {rc['covered_pixel_subframes_per_launch']:.3e} covered (pixel, sub-frame),
{rc['staged_records_per_launch']:.3e} staged records.  Warp efficiency (ncu): K4 {we.get('kernel', float('nan')):.3f} active lanes per
warp instruction; its coverage-test loop runs all 32 lanes ({we.get('coverage_loop_active_lanes', float('nan')):.2f}) but only
{we.get('coverage_loop_useful_lanes', float('nan')):.3f} of the lane tests find a covered pair (census covered / executed).

## Launch list (ncu `gpu__time_duration.sum`, `--clock-control none`; `python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline`)

Cold-cache, serialised per-launch times: compare shares, not absolutes.  `k4_raster_fwd<1,0>` is the
census launch outside the timed region (round 1's kernel with counters); `k_ffma` is the FFMA probe;
`k6_raster_bwd_fx` is the fallback backward over the (image, tile)s the gather listed (none on C4).

{tab_l}

## `ncu --set full` of the raster kernels (C4, one timed step)

{tab_f}

Top stall reasons per source line (`tools/ncu_stalls.py`):

```
{k4s}
{k6s}
```

## History of this round (C4, 1 B200)

{HISTORY}
"""
    open(os.path.join(PROF, "r2e_summary.md"), "w").write(md)
    print("wrote profiles/r2e_summary.md")


if __name__ == "__main__":
    main()
