"""Scratch: k = 0 vs k = 255 (the same pose for 2 full turns) soft gradients at one pixel, GPU vs oracle, soft cut."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import oracle, scenes
from paper_2602_07860_b200 import BlurRenderer
view, py, px = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
sc = scenes.make_c5().subset([view])
delta = 1e-4
dev = torch.device("cuda:0")
v = torch.tensor(np.asarray(sc.verts, np.float32), device=dev)
c = torch.tensor(np.asarray(sc.colors, np.float32), device=dev)
g = np.array([0.0, 0.0, 0.0, 1.0])
G = np.zeros((1, sc.H, sc.W, 4), np.float32); G[0, py, px] = g
res = {}
for k in (0, 255):
    rdv, rdc, rk = oracle.render_bwd(sc, g[None], pixels=[[0, py, px]], delta=delta, sub_range=[[k, k + 1]], want_dkey=True)
    res[("o", k)] = rdv
    for cut in (0.0, 40.0):
        for mc in (0, 1):
            r = BlurRenderer(sc.faces, sc.motion, sc.cams, sc.H, sc.W, sc.V, device=dev, delta=delta, sub_range=[[k, k + 1]],
                             cache_visibility=False, soft_cut=cut, max_chunk=mc)
            r.forward(v, c)
            dv, dc = r.backward(v, c, torch.tensor(G, device=dev), reuse_setup=True)
            dv = dv.cpu().numpy()
            print("k %3d cut %4.0f max_chunk %d |gpu - oracle| %.3e |oracle| %.3e" % (k, cut, mc, np.linalg.norm(dv - rdv), np.linalg.norm(rdv)))
            res[("g", k, cut, mc)] = dv
            del r
print("|oracle k0 - oracle k255| %.3e" % np.linalg.norm(res[("o", 0)] - res[("o", 255)]))
print("|gpu k0 - gpu k255| %.3e" % np.linalg.norm(res[("g", 0, 0.0, 0)] - res[("g", 255, 0.0, 0)]))
d = res[("g", 0, 0.0, 0)] - res[("o", 0)]
idx = np.argsort(np.linalg.norm(d, axis=1))[::-1][:6]
for i in idx:
    print("vertex %d gpu %s oracle %s" % (i, res[("g", 0, 0.0, 0)][i], res[("o", 0)][i]))
