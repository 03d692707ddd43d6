"""Diagnostic: gradient parity breakdown on C4 views."""
import sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
import oracle, scenes
from test_gpu_parity import gpu_render, rel_l2
full = scenes.make_c4()
for imgs in ([2], [11]):
    sc = full.subset(imgs)
    ref = oracle.render_fwd(sc, eps_amb=1e-6)
    G = 2.0 * (ref["rgba"] - sc.target) / ref["rgba"].size
    G2 = G * (~ref["amb_img"])[..., None]
    for name, g in (("all", G), ("non-amb", G2)):
        got = gpu_render(sc, G=g)
        rdv, rdc, rk = oracle.render_bwd(sc, g, want_dkey=True)
        e = np.linalg.norm(got["dv"] - rdv, axis=1)
        worst = np.argsort(-e)[:5]
        print(imgs, name, "amb px", int(ref["amb_img"].sum()), "status", got["status"], "dV rel", rel_l2(got["dv"], rdv),
              "dC rel", rel_l2(got["dc"], rdc), "worst verts", worst, e[worst], "norm", np.linalg.norm(rdv), flush=True)
