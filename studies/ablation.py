#!/usr/bin/env python
"""NEXT-2: the paper's speed comparison (Fig.4) on the B200 -- fast barycentric solver
(per-segment Eq.8 coefficients) vs per-sub-frame solving, forward + gradient in one pass.

Workload (synthetic stand-in for 50 ShapeNet models with ~5,536 faces): icosphere level 4
(5,120 faces) with a seeded low-frequency SH displacement per model, object initialisation
(unit max norm, random rotation about X in [-90, 90] deg), 128x128 front view at
d = 2.232, linear translation x(t) = x0 + (0.5 - t) (A30), N in {10, 25, 50, 100}.
Solvers: 0 fast, 1 naive per-frame set-up (lerp + adjugate per sub-frame, same per-pixel work),
2 naive per-pixel solve (SoftRas-style).  Times: CUDA events around the two raster kernels
(device), and the whole fwd + L2 + bwd call per model (synchronised, includes host overhead).
Prints a markdown table with the least-squares slope (ms per sample)."""
import math
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import scenes  # noqa: E402
from paper_2602_07860_b200 import BlurRenderer  # noqa: E402


def models(n, seed=7):
    rng = np.random.default_rng(seed)
    base, faces = scenes.icosphere(4, 1.0)
    out = []
    for _ in range(n):
        v = scenes.sh_displace(base, rng)
        v = scenes.init_object(v, rng)
        out.append((v.astype(np.float32), rng.uniform(0, 1, (len(v), 3)).astype(np.float32)))
    return faces, out


def main(n_models=20, reps=5):
    faces, ms = models(n_models)
    cam = np.stack([scenes.camera_row(scenes.spherical_eye(scenes.CAM_DIST, 0.0, 0.0))])
    Ns = (10, 25, 50, 100)
    res = {}
    dev = torch.device("cuda")
    for solver in (0, 1, 2):
        for N in Ns:
            mo = scenes.motion_arrays([scenes.translate((-1.0, 0.0, 0.0), N=N)])
            r = BlurRenderer(faces, mo, cam, 128, 128, ms[0][0].shape[0], device=dev, solver=solver)
            tgt = torch.zeros((1, 128, 128, 4), device=dev)
            dev_ms, wall_ms = [], []
            for it in range(reps + 1):
                for v, c in ms:
                    vt, ct = torch.tensor(v, device=dev), torch.tensor(c, device=dev)
                    ef = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                    eb = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                    ef[0].record(); ef[1].record(); eb[0].record(); eb[1].record()
                    torch.cuda.synchronize()
                    t0 = time.perf_counter()
                    out = r.forward(vt, ct, events=ef)
                    loss, g = r.l2_loss_grad(out, tgt)
                    r.backward(vt, ct, g, reuse_setup=True, events=eb)
                    torch.cuda.synchronize()
                    t1 = time.perf_counter()
                    if it > 0:
                        wall_ms.append((t1 - t0) * 1e3)
                        dev_ms.append(ef[0].elapsed_time(ef[1]) + eb[0].elapsed_time(eb[1]))
            res[(solver, N)] = (float(np.mean(dev_ms)), float(np.mean(wall_ms)))
    names = {0: "fast (Eq.8 per-segment coefficients)", 1: "naive per-frame set-up", 2: "naive per-pixel solve"}
    rows = ["| solver | " + " | ".join("N=%d raster ms (call ms)" % N for N in Ns) + " | slope ms/sample (raster) |",
            "|---|" + "---|" * (len(Ns) + 1)]
    slopes = {}
    for solver in (0, 1, 2):
        y = np.array([res[(solver, N)][0] for N in Ns])
        slope = np.polyfit(np.array(Ns, float), y, 1)[0]
        slopes[solver] = slope
        rows.append("| %s | " % names[solver] + " | ".join("%.3f (%.3f)" % res[(solver, N)] for N in Ns) +
                    " | %.5f |" % slope)
    print("\n".join(rows))
    print("\nspeed-up of the fast solver, raster time at N=100: vs per-frame %.2fx, vs per-pixel %.2fx; "
          "slope ratio: %.2fx / %.2fx" % (res[(1, 100)][0] / res[(0, 100)][0], res[(2, 100)][0] / res[(0, 100)][0],
                                          slopes[1] / slopes[0], slopes[2] / slopes[0]))


if __name__ == "__main__":
    main()
