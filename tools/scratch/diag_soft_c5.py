"""Scratch: per-pixel soft gradient comparison (GPU vs oracle) on a C5 view, to find the pixels behind a dV mismatch."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "tests"))
import numpy as np, torch
import oracle, scenes
from paper_2602_07860_b200 import BlurRenderer
view = int(sys.argv[1]) if len(sys.argv) > 1 else 63
sc = scenes.make_c5().subset([view])
delta = 1e-4
dev = torch.device("cuda:0")
r = BlurRenderer(sc.faces, sc.motion, sc.cams, sc.H, sc.W, sc.V, device=dev, delta=delta, cache_visibility=(None if os.environ.get("CACHE", "1") == "1" else False))
v = torch.tensor(np.asarray(sc.verts, np.float32), device=dev)
c = torch.tensor(np.asarray(sc.colors, np.float32), device=dev)
out = r.forward(v, c).cpu().numpy()
a = out[..., 3]
rng = np.random.default_rng(11 + view)
cand = np.argwhere((a > 1e-4) & (a < 0.2))
pick = cand[rng.choice(len(cand), size=min(96, len(cand)), replace=False)]
ref = oracle.render_fwd(sc, pixels=pick, eps_amb=1e-6, delta=delta)
Gp = rng.normal(size=(len(pick), 4)) * (~ref["amb_win"])[:, None]
rows = []
for i in np.nonzero(~ref["amb_win"])[0]:
    G = np.zeros((sc.B, sc.H, sc.W, 4), np.float32)
    G[pick[i, 0], pick[i, 1], pick[i, 2]] = Gp[i]
    out2 = r.forward(v, c)
    dv, dc = r.backward(v, c, torch.tensor(G, device=dev), reuse_setup=True)
    rdv, rdc = oracle.render_bwd(sc, Gp[i:i + 1], pixels=pick[i:i + 1], delta=delta)
    e = np.linalg.norm(dv.cpu().numpy() - rdv)
    rows.append((e, np.linalg.norm(rdv), i, tuple(pick[i]), float(ref["rgba"][i, 3]), Gp[i].tolist()))
rows.sort(reverse=True)
tot = np.sqrt(sum(x[1] ** 2 for x in rows))
print("total ref norm %.3e" % tot)
for e, n, i, p, al, g in rows[:8]:
    print("pixel %s alpha %.4g |err| %.3e |ref| %.3e G %s" % (p, al, e, n, np.round(g, 3)))
