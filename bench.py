#!/usr/bin/env python
"""Benchmark of the hot path: one inverse-rendering step (fwd -> L2 loss -> bwd -> all-reduce) of
the motion-blur rasterizer on N GPUs of one node; prints ONE JSON line (rank 0).

  python bench.py [--gpus N --steps K --warmup W] [--config C4] [--impl reference]
  torchrun --nproc-per-node N bench.py --gpus N ...        (one process per GPU, NCCL)

Workload (BASELINE.json configs[3], "C4"): 10,242-vertex / 20,480-face genus-0 mesh (icosphere
level 5 template; targets = renders of its seeded SH-displaced version), 16 observed 512x512
images (8 translational, 8 rotational views), N = 100 sub-frames, S = 1 / 12 segments; images
sharded over ranks, NCCL all-reduce of [dV || dC].  Synthetic, seeded (scenes/).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "blurred images/s (fwd+bwd)"
UNIT = "images/s"
# FP32 SIMT peak derived from the profiling guide's unit counts and clock:
# 148 SMs x 128 FP32 lanes x 2 flop (FFMA) x 1.965 GHz
FP32_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12
# algorithmic work per unit: flop per covered (pixel, face, sub-frame) pair,
# per covered (pixel, sub-frame) shade, per (face, sub-frame) coefficient evaluation, and the
# backward's extra work per covered (pixel, sub-frame)
FLOP_PAIR, FLOP_SHADE, FLOP_SETUP, FLOP_BWD = 18.0, 25.0, 30.0, 100.0
# soft background coverage (NEXT-1): flop per evaluated (pixel, face, sub-frame) term (census [4]: the
# terms K8 evaluates, within 18 delta: the default cut-off of both kernels)
# in the forward
# (w1, w2: 8; three projections + quadratic forms: 3 x 12; Eq.14 form + exp + product: 10) and in
# the backward (pass 1 the same, pass 2 the same + 16 for the gradient and its keyframe split; with
# the visibility cache K9 reads K8's products and runs pass 2 only: 70)
FLOP_SOFT_FWD, FLOP_SOFT_BWD, FLOP_SOFT_BWD_CACHED = 54.0, 124.0, 70.0
LAUNCHES_FWD, LAUNCHES_LOSS, LAUNCHES_BWD = 9, 1, 2
LAUNCHES_SOFT_FWD, LAUNCHES_SOFT_BWD = 9, 2     # soft bins (7) + K8 + reduce; K9C (cached products) + K9


def _free_port() -> int:
    import socket
    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    p = so.getsockname()[1]
    so.close()
    return p


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--config", default="C4")
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--split", type=int, default=0, help="sub-frame ranges per image (0 = auto)")
    p.add_argument("--max-chunk", type=int, default=0)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=12.0, help="target CPU time of the oracle sample")
    p.add_argument("--ref-images", type=int, default=2, help="--impl reference: images per timed step")
    p.add_argument("--graph", action="store_true",
                   help="replay the step as a CUDA graph (launch-bound configs C1-C3; 1 GPU, no sub-frame split)")
    p.add_argument("--delta", type=float, default=0.0,
                   help="soft background coverage bandwidth (NEXT-1, Eq.10-15; the paper uses 1e-4); 0 = hard path")
    return p.parse_args()


# ------------------------------------------------------------------ helpers

class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region (B200_PROFILING.md)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.path = os.path.join("/tmp", "bench_clocks_%d_%d.csv" % (os.getpid(), gpu_index))

    def start(self):
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), "--query-gpu=" + self.Q,
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.fh.close()
        sm, smax, reasons = [], [], set()
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def make_target(sc, dev, delta=0.0):
    """Loss targets: renders of the displaced mesh (C4/C5 inverse-rendering step) or the seeded
    uniform targets (C1-C3).  Built before timing."""
    import torch
    if "displaced_verts" not in sc.meta:
        return torch.tensor(sc.target, device=dev)
    from paper_2602_07860_b200 import BlurRenderer
    out = torch.empty((sc.B, sc.H, sc.W, 4), dtype=torch.float32, device=dev)
    for b0 in range(0, sc.B, 8):
        sub = sc.subset(list(range(b0, min(sc.B, b0 + 8))))
        r = BlurRenderer(sub.faces, sub.motion, sub.cams, sub.H, sub.W, sub.V, device=dev, delta=delta)
        r.forward(torch.tensor(sc.meta["displaced_verts"], device=dev), torch.tensor(sc.colors, device=dev),
                  out=out[b0:b0 + sub.B])
        del r
    torch.cuda.synchronize()
    return out


def cpu_baseline(sc, target_seconds: float, delta: float = 0.0):
    """Time the fp64 oracle (as it stands) fwd + bwd on a bounded sample of the same workload, all
    host cores: whole images (translational and rotational views alternately) until about
    `target_seconds` of CPU time, or a leading sub-frame range of one image if a single image
    already takes longer.  Returns images/s and the sample description."""
    import oracle
    cores = oracle.num_threads(0)
    N = int(sc.motion["n_sub"][0])
    order = []
    lo, hi = 0, sc.B - 1
    while lo <= hi:                       # 0, B-1, 1, B-2, ... (both motion kinds)
        order.append(lo)
        if hi != lo:
            order.append(hi)
        lo, hi = lo + 1, hi - 1

    def run(imgs, ks):
        sub = sc.subset(imgs)
        rng = [[0, ks]] * sub.B
        t0 = time.perf_counter()
        fw = oracle.render_fwd(sub, sub_range=rng, delta=delta)
        G = 2.0 * (fw["rgba"] - (sub.target if sub.target is not None else 0.0)) / fw["rgba"].size
        oracle.render_bwd(sub, G, sub_range=rng, delta=delta)
        return time.perf_counter() - t0

    t1 = run(order[:1], N)                 # one whole image
    ks, reps = N, 1
    if t1 >= target_seconds:
        imgs, t = order[:1], t1
    else:
        imgs = sorted(order[:max(1, min(sc.B, int(target_seconds / t1)))])
        if len(imgs) == 1:                   # tiny workloads: repeat the sample
            reps = max(1, min(1000, int(target_seconds / max(t1, 1e-6))))
            t = sum(run(imgs, N) for _ in range(reps))
        else:
            t = run(imgs, ks)
    images = len(imgs) * reps
    return {"value": images / t, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": "fp64 oracle (binned%s) fwd+bwd of %d of %d images of %s (%s) x %d repetitions, all %d "
                      "sub-frames: %.1f s on %d threads" % (", soft delta=%g" % delta if delta > 0 else "", len(imgs),
                                                             sc.B, sc.name, imgs, reps, N, t, cores),
            "seconds": t}


def workload_config(sc, args, world, split_groups=False, graph=False):
    """The `config` object of the JSON line (both arms)."""
    soft = args.delta > 0
    return {"workload": sc.name, "images": sc.B, "H": sc.H, "W": sc.W, "faces": sc.F, "vertices": sc.V,
            "subframes": int(sc.motion["n_sub"][0]), "segments": sorted({int(x) for x in sc.motion["n_seg"]}),
            **({"delta": args.delta, "coverage": "soft (Eq.10-15)"} if soft else {}),
            "parallelism": "image-sharded x%d" % world + (" + subframe split" if split_groups else ""),
            "l2": "flushed (256 MB write) before every timed step",
            **({"cuda_graph": True} if graph else {})}


def run_reference(args, rank, world, out_json):
    """The reference arm: the fp64 CPU oracle as it stands (binned, all host cores), one bounded sample
    of the workload per step -- `sample_images` whole images (translational and rotational views in
    turn), fwd + bwd, all sub-frames -- timed step by step.  ms_per_step is the measured time of one
    such step; value = images processed / time."""
    if rank != 0:
        return
    import oracle
    import scenes
    sc = scenes.make(args.config)
    cores = oracle.num_threads(0)
    order = []
    lo, hi = 0, sc.B - 1
    while lo <= hi:                       # 0, B-1, 1, B-2, ... (both motion kinds)
        order.append(lo)
        if hi != lo:
            order.append(hi)
        lo, hi = lo + 1, hi - 1
    m = max(1, min(sc.B, args.ref_images))
    N = int(sc.motion["n_sub"][0])
    times, pos = [], 0
    for it in range(args.warmup + args.steps):
        imgs = sorted(order[(pos + i) % len(order)] for i in range(m))
        pos += m
        sub = sc.subset(imgs)
        t0 = time.perf_counter()
        fw = oracle.render_fwd(sub, delta=args.delta)
        G = 2.0 * (fw["rgba"] - (sub.target if sub.target is not None else 0.0)) / fw["rgba"].size
        oracle.render_bwd(sub, G, delta=args.delta)
        if it >= args.warmup:
            times.append(time.perf_counter() - t0)
    tot = sum(times)
    v = m * len(times) / tot
    sample = ("fp64 oracle (binned%s) fwd+bwd of %d of the %d images of %s per step (all %d sub-frames), %d "
              "timed steps: %.1f s on %d threads" % (", soft delta=%g" % args.delta if args.delta > 0 else "", m,
                                                    sc.B, sc.name, N, len(times), tot, cores))
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * tot / len(times),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": workload_config(sc, args, world),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), file=out_json, flush=True)


# ------------------------------------------------------------------ main (ours)

def _stdout_to_stderr():
    """Route file descriptor 1 to stderr for the run (NCCL and CUDA libraries print banners on stdout)
    and return a writer for the real stdout, which receives the one JSON line."""
    real = os.dup(1)
    sys.stdout.flush()
    os.dup2(2, 1)
    return os.fdopen(real, "w")


def main():
    args = parse()
    out_json = _stdout_to_stderr()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world, out_json)
        return
    import torch
    import torch.distributed as dist

    import scenes
    from paper_2602_07860_b200 import BlurRenderer, _lib
    from paper_2602_07860_b200.renderer import cache_bytes_per_image
    from paper_2602_07860_b200.dist import ShardedStep

    assert torch.cuda.is_available(), "bench.py needs CUDA"
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # NCCL at every world size (a 1-rank group at N = 1): the timed step is the same product path,
    # ShardedStep with its [dV || dC || loss] all-reduce, on one GPU and on eight
    os.environ.setdefault("NCCL_DEBUG", "WARN")     # no version banner on stdout (one JSON line)
    if world == 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(_free_port()))
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
    dist.init_process_group("nccl", device_id=dev)
    sc = scenes.make(args.config)
    target = make_target(sc, dev, args.delta)
    verts = torch.tensor(sc.verts, device=dev)
    colors = torch.tensor(sc.colors, device=dev)

    def make_renderer(images, sub_range, workspace=None):
        s = sc.subset(images)
        return BlurRenderer(s.faces, s.motion, s.cams, s.H, s.W, s.V, device=dev, sub_range=sub_range,
                            max_chunk=args.max_chunk, delta=args.delta, workspace=workspace)

    # whole images in passes whose backward winner index fits the cache budget (C5: 2 images per pass)
    per_image = cache_bytes_per_image(sc.H, sc.W, int(max(sc.motion["n_sub"])), args.delta)
    pass_images = max(1, BlurRenderer.CACHE_BUDGET_BYTES // per_image) if not args.graph else 0
    step = ShardedStep(sc.motion["n_sub"], target, make_renderer, rank, world, split=args.split, device=dev,
                       reduce=True, pass_images=pass_images)
    rend = step.renderer
    stream = torch.cuda.current_stream()

    # census (outside timing): algorithmic unit counts of this rank's forward
    census = torch.zeros(12, dtype=torch.int64, device=dev)
    units = np.zeros(12)
    if rend is not None:
        step.census(verts, colors, census)
        units = census.cpu().numpy().astype(np.float64)
    n_fsub = float(sum(u.k1 - u.k0 for u in step.mine)) * sc.F      # (face, sub-frame) evaluations

    # raster-kernel timing events (recorded inside the C-ABI calls on this stream)
    def evpair():
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        b.record(stream)
        return a, b

    flush_buf = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)   # 256 MB > 126 MB L2

    def one_step(ev_f=None, ev_b=None, ev_sf=None, ev_sb=None):
        # events: lists of CUDA event pairs, one per pass
        ev = {"fwd": ev_f, "bwd": ev_b, "soft_fwd": ev_sf, "soft_bwd": ev_sb} if ev_f is not None else None
        loss, dv, dc = step(verts, colors, events=ev)
        return loss

    graph = None
    if args.graph:
        if rend is None or step.groups or world > 1 or step.n_passes > 1:
            raise SystemExit("--graph needs 1 GPU and no sub-frame split")
        graph = rend.capture_step(verts, colors, step.targets, n_norm=step.n_norm)

    def timed_step(ev_f=None, ev_b=None, ev_sf=None, ev_sb=None):
        if graph is None:
            return one_step(ev_f, ev_b, ev_sf, ev_sb)
        loss, dv, dc, _ = graph.replay()
        return loss

    for _ in range(max(3, args.warmup)):
        timed_step()
    torch.cuda.synchronize()
    if rend is not None:
        st = rend.status()
        if st & 3:
            raise RuntimeError("device status %d after warm-up" % st)

    K = args.steps
    ev_s = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    ev_e = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    npass = step.n_passes
    evf = [[evpair() for _ in range(npass)] for _ in range(K)]
    evb = [[evpair() for _ in range(npass)] for _ in range(K)]
    soft = args.delta > 0
    evsf = [[evpair() for _ in range(npass)] if soft else None for _ in range(K)]
    evsb = [[evpair() for _ in range(npass)] if soft else None for _ in range(K)]
    clocks = ClockSampler(local)
    dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.3)
    for i in range(K):
        flush_buf.zero_()                                       # L2 flush between timed steps
        ev_s[i].record(stream)
        timed_step(evf[i], evb[i], evsf[i], evsb[i])
        ev_e[i].record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    clk = clocks.stop()
    step_ms = [ev_s[i].elapsed_time(ev_e[i]) for i in range(K)]
    tot_ms = float(sum(step_ms))
    if graph is not None:   # kernel events are not part of the graph: time the kernels in eager steps
        for i in range(K):
            flush_buf.zero_()
            one_step(evf[i], evb[i], evsf[i], evsb[i])
        torch.cuda.synchronize()
    def span(pairs):   # summed over the passes of a step
        return sum(a.elapsed_time(b) for a, b in pairs)
    fwd_ms = [span(evf[i]) for i in range(K)] if rend is not None else [0.0]
    bwd_ms = [span(evb[i]) for i in range(K)] if rend is not None else [0.0]
    sf_ms = [span(evsf[i]) for i in range(K)] if soft and rend is not None else [0.0]
    sb_ms = [span(evsb[i]) for i in range(K)] if soft and rend is not None else [0.0]
    t = torch.tensor([tot_ms], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    tot_max = float(t.item())
    ms_per_step = tot_max / K
    value = sc.B / (ms_per_step / 1000.0)

    # roofline of the dominant kernel (raster fwd K4 or raster bwd K6), this rank's launches
    nec, cov, cand_all, staged_all, soft_terms, soft_staged, soft_items, soft_iters = units[:8]
    # the timed forward's own counts (census [8..11], same order as [0..3]): it skips the lists of faces turned
    # away from the camera where every pixel already has a nearer winner, so it executes fewer tests than every
    # bin face at its footprints (cand_all); round 1's kernel (no skip) leaves them 0 -> the full counts
    cand, cov_exec, staged = (units[10], units[8], units[11]) if units[10] > 0 else (cand_all, nec, staged_all)
    fw_flop = FLOP_PAIR * nec + FLOP_SHADE * cov + FLOP_SETUP * n_fsub
    # K6 with the visibility buffer (BlurRenderer default) does not recompute the forward's tests
    bw_flop = (FLOP_BWD * cov + FLOP_SETUP * n_fsub) if (rend is not None and rend.cache_flags) else \
        fw_flop + FLOP_BWD * cov
    f_avg, b_avg = float(np.mean(fwd_ms)), float(np.mean(bwd_ms))
    # the timed kernels: K4 = k4l_raster_fwd (lean forward); K6 = k6v_raster_bwd (visibility gather) with the
    # cache, k6_raster_bwd_fx (recomputed visibility) without
    cached = rend is not None and bool(rend.cache_flags)
    kernels = [("k4l_raster_fwd", fw_flop, f_avg), ("k6v_raster_bwd" if cached else "k6_raster_bwd_fx", bw_flop, b_avg)]
    if soft:
        kernels += [("k8_soft_fwd", FLOP_SOFT_FWD * soft_terms, float(np.mean(sf_ms))),
                    ("k9_soft_bwd", (FLOP_SOFT_BWD_CACHED if (rend is not None and rend.cache_flags) else FLOP_SOFT_BWD) * soft_terms,
                     float(np.mean(sb_ms)))]
    kname, flop, dur = max(kernels, key=lambda k: k[2])
    achieved = flop / (dur / 1000.0) / 1e12 if dur > 0 else 0.0
    traffic, prof = None, {}
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        try:
            prof = json.load(open(tp)).get(sc.name, {})
            traffic = prof.get(kname)
        except Exception:
            traffic, prof = None, {}
    hbm_peak, hbm_src = 6546.2, "MEASURED_PEAKS.json hbm_gbs (round 1 copy of the file)"
    try:
        hbm_peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
        hbm_src = "MEASURED_PEAKS.json hbm_gbs"
    except Exception:
        pass
    # HBM side of the same kernel: the DRAM bytes ncu measured per launch over its live duration, and
    # the algorithmic bytes (16 B/px written by the forward, 48 B/px read+written by loss
    # and backward)
    n_px = float(len(step.images)) * sc.H * sc.W
    alg_bytes = (16.0 if kname.startswith(("k4", "k8")) else 48.0) * n_px
    hbm = {"dram_bytes_per_launch": traffic, "algorithmic_bytes_per_launch": alg_bytes, "peak_gbs": hbm_peak,
           "peak_source": hbm_src,
           "achieved_gbs": (traffic / (dur / 1000.0) / 1e9) if (traffic and dur > 0) else None}
    hbm["frac"] = hbm["achieved_gbs"] / hbm_peak if hbm["achieved_gbs"] else None
    wp = prof.get("warp_efficiency", {}).get(kname) or {}
    # the coverage loop walks a warp-uniform face mask, so its lanes are all active (ncu); the share of
    # them whose test covers its pixel is the useful-lane efficiency (census, this run)
    weff = {"kernel": wp.get("kernel"), "coverage_loop_active_lanes":
            None if wp.get("coverage_loop") is None else min(1.0, wp["coverage_loop"]),
            "coverage_loop_useful_lanes": (cov_exec / cand) if cand else None,
            "source": "ncu --set full (profiles/traffic.json) for the active lanes; census covered / executed "
                      "tests for the useful ones"}
    roofline = {"bound": "alu", "kernel": kname, "achieved": achieved, "peak": FP32_PEAK_TFLOPS,
                "unit": "TFLOP/s", "frac": achieved / FP32_PEAK_TFLOPS, "traffic": traffic,
                "hbm_frac": hbm["frac"], "hbm": hbm,
                # active lanes per executed warp instruction / 32 (ncu, profiles/traffic.json): the whole
                # kernel and its coverage-test loop
                "warp_efficiency": weff,
                "peak_source": "derived: 148 SM x 128 FP32 lanes x 2 x 1.965 GHz (B200_PROFILING.md nominal "
                               "SM count and clocks.max.sm)",
                "fwd_raster_ms": f_avg, "bwd_raster_ms": b_avg,
                **({"soft_fwd_ms": float(np.mean(sf_ms)), "soft_bwd_ms": float(np.mean(sb_ms))} if soft else {}),
                "executed_pair_tests_per_launch": cand, "all_faces_pair_tests_per_launch": cand_all,
                "covered_among_executed_per_launch": cov_exec, "necessary_pairs_per_launch": nec,
                "covered_pixel_subframes_per_launch": cov, "staged_records_per_launch": staged,
                # every timed kernel: algorithmic TFLOP/s (same per-unit figures) and fraction of the peak
                "kernels_frac": {k[0]: (k[1] / (k[2] / 1000.0) / 1e12 / FP32_PEAK_TFLOPS if k[2] > 0 else 0.0)
                                 for k in kernels},
                **({"soft_terms_per_launch": soft_terms, "soft_staged_records_per_launch": soft_staged,
                    "soft_items_per_launch": soft_items, "soft_face_iterations_per_launch": soft_iters,
                    "kernels_ms": {k[0]: k[2] for k in kernels}} if soft else {})}

    # measured FFMA throughput (context for the derived peak)
    ffma = None
    if rank == 0:
        sink = torch.empty(148 * 8 * 256, dtype=torch.float32, device=dev)
        _lib.blur_ffma_probe(148 * 8, 64, sink)
        torch.cuda.synchronize()
        best = 0.0
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fl = _lib.blur_ffma_probe(148 * 8, 512, sink)
            b.record(stream)
            torch.cuda.synchronize()
            best = max(best, fl / (a.elapsed_time(b) / 1000.0) / 1e12)
        ffma = best

    # end-to-end through the public API with host buffers (pinned), copies inside the timed region
    e2e = None
    if not args.no_e2e and rend is not None:
        h_verts = torch.tensor(sc.verts).pin_memory()
        h_cols = torch.tensor(sc.colors).pin_memory()
        h_tgt = step.targets.cpu().pin_memory()
        d_verts, d_cols, d_tgt = torch.empty_like(verts), torch.empty_like(colors), torch.empty_like(step.targets)
        h_out = torch.empty(6 * sc.V + 1, dtype=torch.float32).pin_memory()
        saved = step.targets

        copy_stream = torch.cuda.Stream(device=dev)
        tgt_ready = torch.cuda.Event()

        def e2e_step():
            d_verts.copy_(h_verts, non_blocking=True)
            d_cols.copy_(h_cols, non_blocking=True)
            # the observed images go up on a copy stream, overlapped with the forward pass; the
            # copy waits for the previous step's use of the buffer, the loss waits for the copy
            copy_stream.wait_stream(stream)
            with torch.cuda.stream(copy_stream):
                d_tgt.copy_(h_tgt, non_blocking=True)
                tgt_ready.record(copy_stream)
            step.targets = d_tgt
            flat = one_step_public(d_verts, d_cols)
            h_out.copy_(flat, non_blocking=True)

        def one_step_public(v, c):
            loss, dv, dc = step(v, c, targets_ready=tgt_ready)
            return torch.cat([dv.reshape(-1), dc.reshape(-1), loss])

        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize()
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(K):
            e2e_step()
        b.record(stream)
        torch.cuda.synchronize()
        te = torch.tensor([a.elapsed_time(b)], dtype=torch.float64, device=dev)
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        step.targets = saved
        e2e = {"value": sc.B / (float(te.item()) / K / 1000.0), "unit": UNIT,
               "h2d_bytes_per_step": int(h_verts.numel() * 4 + h_cols.numel() * 4 + h_tgt.numel() * 4),
               "d2h_bytes_per_step": int(h_out.numel() * 4)}

    cb = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = cpu_baseline(sc, args.cpu_seconds, args.delta)
        cb.pop("seconds", None)

    if rank == 0:
        n_sub = int(sc.motion["n_sub"][0])
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
                "warmup": max(3, args.warmup), "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": {**workload_config(sc, args, world, bool(step.groups), graph is not None),
                           **({"passes_per_rank": step.n_passes,
                               "visibility_cache": "per pass, <= %d MiB (a one-image pass: <= %d MiB)"
                                                   % (BlurRenderer.CACHE_BUDGET_BYTES >> 20,
                                                      BlurRenderer.CACHE_IMAGE_BYTES >> 20)}
                              if step.n_passes > 1 else {})},
                "barycentric_evals_per_s": {"executed": cand * world / (ms_per_step / 1000.0),
                                            "necessary": nec * world / (ms_per_step / 1000.0),
                                            "note": "per-rank census x ranks (rank 0's counts)"},
                "roofline": roofline, "ffma_measured_tflops": ffma, "clocks": clk,
                "gpu_launches": (LAUNCHES_FWD + LAUNCHES_LOSS + LAUNCHES_BWD +
                                 (LAUNCHES_SOFT_FWD + LAUNCHES_SOFT_BWD if soft else 0)) * K,
                "e2e": e2e, "cpu_baseline": cb}
        print(json.dumps(line), file=out_json, flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
