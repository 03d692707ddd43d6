"""Diagnostic (not a test): localise GPU/oracle mismatches on a config."""
import sys

import numpy as np

sys.path.insert(0, "."); sys.path.insert(0, "tests")
import oracle  # noqa: E402
import scenes  # noqa: E402
from test_gpu_parity import gpu_render  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
sc = scenes.make(name).subset([0, 1])
ref = oracle.render_fwd(sc, eps_amb=1e-6)
for G, bf in [(0, 0.0), (1, 0.0), (16, 0.0), (0, 1e-9)]:
    got = gpu_render(sc, max_chunk=G, bin_factor=bf)
    err = np.abs(got["rgba"] - ref["rgba"]).max(-1)
    err[ref["amb_img"]] = 0
    bad = np.argwhere(err > 1e-4)
    print("G", G, "bf", bf, "status", got["status"], "nbad", len(bad), "max", err.max())
    if G == 0 and bf == 0.0:
        bad0 = bad
for (b, j, i) in bad0[:6]:
    N = int(sc.motion["n_sub"][b])
    pix = np.array([[b, j, i]], np.int32)
    row = []
    for k in range(N):
        o = oracle.render_fwd(sc, pixels=pix, ids_k=k)["ids"][0]
        g = gpu_render(sc.subset([b]), ids_k=k)["ids"][0, j, i]
        if o != g:
            row.append((k, int(o), int(g)))
    print("pixel", (b, j, i), "err", err[b, j, i] if False else "", "mismatch k (oracle, gpu):", row[:8])
    if row:
        k, fo, fg = row[0]
        key, valid, Q = oracle.keyframes(sc, b)
        s_, t_ = oracle.schedule(N, int(sc.motion["n_seg"][b]))
        s, tau = s_[k], t_[k]
        g = (1 - tau) * key[s] + tau * key[s + 1]
        u = -1 + (2 * i + 1) / sc.W
        v = 1 - (2 * j + 1) / sc.H
        for f in (fo, fg):
            if f < 0:
                continue
            fv = sc.faces[f]
            F = np.array([g[fv, 0], g[fv, 1], np.ones(3)])
            w = np.linalg.solve(F, [u, v, 1])
            print("   face", f, "w", w, "z", w @ g[fv, 2], "det", np.linalg.det(F), "verts", fv)
