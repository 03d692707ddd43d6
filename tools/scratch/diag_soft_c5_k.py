"""Scratch: per-sub-frame soft gradient at one pixel of a C5 view (GPU vs oracle)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import oracle, scenes
from paper_2602_07860_b200 import BlurRenderer
view, py, px = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
sc = scenes.make_c5().subset([view])
delta = 1e-4
dev = torch.device("cuda:0")
N = int(sc.motion["n_sub"][0])
v = torch.tensor(np.asarray(sc.verts, np.float32), device=dev)
c = torch.tensor(np.asarray(sc.colors, np.float32), device=dev)
g = np.array([0.0, 0.0, 0.0, 1.0])
G = np.zeros((1, sc.H, sc.W, 4), np.float32); G[0, py, px] = g
rows = []
ks = range(N) if len(sys.argv) < 5 else [int(k) for k in sys.argv[4].split(",")]
for k in ks:
    r = BlurRenderer(sc.faces, sc.motion, sc.cams, sc.H, sc.W, sc.V, device=dev, delta=delta, sub_range=[[k, k + 1]], cache_visibility=False)
    out = r.forward(v, c)
    a_gpu = float(out[0, py, px, 3])
    dv, dc = r.backward(v, c, torch.tensor(G, device=dev), reuse_setup=True)
    ref = oracle.render_fwd(sc, pixels=[[0, py, px]], delta=delta, sub_range=[[k, k + 1]], eps_amb=1e-6)
    rdv, rdc = oracle.render_bwd(sc, g[None], pixels=[[0, py, px]], delta=delta, sub_range=[[k, k + 1]])
    e = np.linalg.norm(dv.cpu().numpy() - rdv)
    rows.append((e, k, np.linalg.norm(rdv), a_gpu, float(ref["rgba"][0, 3]), bool(ref["amb_win"][0])))
    del r
rows.sort(reverse=True)
for e, k, n, ag, ao, amb in rows[:10]:
    print("k %3d |err| %.3e |ref| %.3e alpha gpu %.6g oracle %.6g amb %d" % (k, e, n, ag * N, ao * N, amb))
