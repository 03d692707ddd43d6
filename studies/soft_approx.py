#!/usr/bin/env python
"""NEXT-1 study: how far the paper's endpoint approximation (Eq.13: closest point computed on the
keyframe triangle F(X), X = [tau > 0.5]) is from the exact closest point on F(tau) (Eq.12), on the
B200, for the soft alpha of whole blurred images.  The paper calls the difference "minor
approximation errors" without a number.  Workloads: C2 (translation) and C3/C4 views
(rotation with 24 / 12 segments), delta = 1e-4.  Reports max / mean |alpha_13 - alpha_12|
over pixels and the time of the soft kernels for both."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import scenes  # noqa: E402
from paper_2602_07860_b200 import BlurRenderer  # noqa: E402


def soft_ms(r, v, c, reps=5):
    ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    ev[0].record()   # mark as recorded for torch; the C ABI re-records them around the soft kernel
    ev[1].record()
    r.forward(v, c)
    ts = []
    for _ in range(reps):
        out = r.forward(v, c, soft_events=ev)
        torch.cuda.synchronize()
        ts.append(ev[0].elapsed_time(ev[1]))
    return out, float(np.median(ts))


def main():
    dev = torch.device("cuda:0")
    print("# Soft coverage: Eq.13 endpoint approximation vs Eq.12 exact closest point (B200, round 1)\n")
    print("`python studies/soft_approx.py`, delta = 1e-4.  alpha differences over all pixels of the blurred images.\n")
    print("| workload | motion | max abs d-alpha | mean abs d-alpha (pixels with alpha in (0,1)) | K8 ms Eq.13 | K8 ms Eq.12 |")
    print("|---|---|---|---|---|---|")
    for name, imgs in [("C2", [0, 1, 2, 3]), ("C3", [0, 2, 4, 6]), ("C4", [0, 3, 8, 12])]:
        sc = scenes.make(name).subset(imgs)
        v, c = torch.tensor(sc.verts, device=dev), torch.tensor(sc.colors, device=dev)
        outs, ts = [], []
        for exact in (False, True):
            r = BlurRenderer(sc.faces, sc.motion, sc.cams, sc.H, sc.W, sc.V, device=dev, delta=1e-4, soft_exact=exact)
            o, t = soft_ms(r, v, c)
            outs.append(o[..., 3].cpu().numpy())
            ts.append(t)
        d = np.abs(outs[0] - outs[1])
        band = (outs[1] > 0) & (outs[1] < 1)
        kinds = sorted({int(k) for k in sc.motion["kind"]})
        mot = "/".join({1: "translation", 2: "rotation", 3: "parabolic"}[k] for k in kinds)
        print("| %s (%d x %d^2) | %s | %.4f | %.2e | %.2f | %.2f |" % (name, sc.B, sc.H, mot, d.max(), d[band].mean(),
                                                                    ts[0], ts[1]))
    print("\nWere F(tau) a pure screen-space shift of F(X), Eq.13 would be exact (p' = p - shift); the perspective"
          " projection of a 3D translation also scales the triangle (C2's motion has a depth component), and a"
          " rotation within a segment changes its shape, so the closest point moves and so does alpha.  The"
          " approximation costs nothing measurable: both variants run in the same time.")


if __name__ == "__main__":
    main()
