"""Check (GPU): K8 with its 18-delta cut gives bit-identical soft alpha and products to K8 with the
full cut (variant build BR_K8_CUT=1e30f).  usage: python tools/k8_cut_check.py LIB_A LIB_B [CFG]"""
import os
import subprocess
import sys

import numpy as np

if len(sys.argv) > 3 and sys.argv[1] == "--one":
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import scenes
    from paper_2602_07860_b200 import BlurRenderer
    sc = scenes.make(sys.argv[3])
    dev = torch.device("cuda:0")
    r = BlurRenderer(sc.faces, sc.motion, sc.cams, sc.H, sc.W, sc.V, device=dev, delta=1e-4)
    v = torch.tensor(np.asarray(sc.verts, np.float32), device=dev)
    c = torch.tensor(np.asarray(sc.colors, np.float32), device=dev)
    out = r.forward(v, c).cpu().numpy()
    g = torch.tensor(np.random.default_rng(0).normal(size=out.shape).astype(np.float32) * 1e-4, device=dev)
    dv, dc = r.backward(v, c, g, reuse_setup=True)
    np.savez(sys.argv[2], rgba=out, dv=dv.cpu().numpy(), dc=dc.cpu().numpy())
    sys.exit(0)
cfg = sys.argv[3] if len(sys.argv) > 3 else "C3"
res = []
for i, lib in enumerate(sys.argv[1:3]):
    f = "/tmp/k8cut_%d.npz" % i
    subprocess.check_call([sys.executable, __file__, "--one", f, cfg], env=dict(os.environ, BLURRAST_LIB=os.path.abspath(lib)))
    res.append(np.load(f))
a, b = res
print(cfg, "rgba bit-identical:", np.array_equal(a["rgba"], b["rgba"]),
      "max |diff| %g" % np.abs(a["rgba"] - b["rgba"]).max(),
      "dv rel %g" % (np.linalg.norm(a["dv"] - b["dv"]) / np.linalg.norm(b["dv"])))
d = np.abs(a["rgba"] - b["rgba"])
print("channels max diff", d.reshape(-1, 4).max(0), "pixels > 1e-6:", int((d.max(-1) > 1e-6).sum()))
for idx in np.argsort(d.max(-1).ravel())[::-1][:5]:
    bi, y, x = np.unravel_index(idx, d.shape[:3])
    print((bi, y, x), a["rgba"][bi, y, x], b["rgba"][bi, y, x])
