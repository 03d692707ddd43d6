#!/usr/bin/env python
"""NEXT-3 / Appendix 'Segmentation Analysis' on the B200: PSNR of piecewise-linear
(S-segment) rotation blur against the exact-pose blur of the same N sub-frames.

Workload: the C3 spinning top (synthetic stand-in for the paper's Spot model),
one full turn about +y (A31), 512x512, N = 240 sub-frames.  The exact-pose reference renders every
sub-frame at its exact rigid pose (N-1 segments).  Prints a markdown table."""
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import scenes  # noqa: E402
from paper_2602_07860_b200 import BlurRenderer  # noqa: E402


def render(sc, motion):
    mo = scenes.motion_arrays([motion] * sc.B)
    r = BlurRenderer(sc.faces, mo, sc.cams, sc.H, sc.W, sc.V)
    out = r.forward(torch.tensor(sc.verts, device="cuda"), torch.tensor(sc.colors, device="cuda"))
    torch.cuda.synchronize()
    return out.cpu().numpy()


def psnr(a, b):
    mse = float(np.mean((a[..., :3] - b[..., :3]) ** 2))
    return 10 * math.log10(1.0 / max(mse, 1e-30))


def main():
    sc = scenes.make_c3().subset([0, 2, 4])
    N = 240
    rot = dict(axis=(0, 1, 0), angle=2 * math.pi)
    ref = render(sc, scenes.exact_pose(scenes.rotate(rot["axis"], rot["angle"], N=N, S=1)))
    rows = ["| segments | schedule | samples | PSNR vs exact pose (dB) |", "|---|---|---|---|"]
    for S in (6, 12, 24, 48):
        img = render(sc, scenes.rotate(rot["axis"], rot["angle"], N=N, S=S))
        rows.append("| %d | GLOBAL_INCLUSIVE | %d | %.2f |" % (S, N, psnr(img, ref)))
    for S, K in ((6, 40), (12, 20), (24, 10), (48, 5)):
        img = render(sc, scenes.rotate(rot["axis"], rot["angle"], N=S * K, S=S, rule=scenes.PAPER_SEGMENTED))
        rows.append("| %d | PAPER_SEGMENTED %dx%d | %d | %.2f |" % (S, S, K, S * K, psnr(img, ref)))
    print("\n".join(rows))


if __name__ == "__main__":
    main()
