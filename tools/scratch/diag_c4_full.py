"""Scratch: locate the worst non-ambiguous pixel of the full C4 batch (GPU vs oracle) and compare it per sub-frame."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import oracle, scenes
from paper_2602_07860_b200 import BlurRenderer
sc = scenes.make_c4()
dev = torch.device("cuda:0")
cache = os.environ.get("CACHE", "1") == "1"
r = BlurRenderer(sc.faces, sc.motion, sc.cams, sc.H, sc.W, sc.V, device=dev, cache_visibility=cache)
v = torch.tensor(np.asarray(sc.verts, np.float32), device=dev)
c = torch.tensor(np.asarray(sc.colors, np.float32), device=dev)
out = r.forward(v, c).cpu().numpy()
ref = oracle.render_fwd(sc, eps_amb=1e-6)
err = np.abs(out - ref["rgba"])
err[ref["amb_img"]] = 0
flat = np.argsort(err.max(-1).ravel())[::-1][:6]
for fi in flat:
    b, y, x = np.unravel_index(fi, err.shape[:3])
    print("view %d pixel (%d, %d) err %.3g gpu %s ref %s amb_win %d" % (b, y, x, err[b, y, x].max(), out[b, y, x], ref["rgba"][b, y, x], ref["amb_win"][b, y, x]))
b, y, x = np.unravel_index(flat[0], err.shape[:3])
one = sc.subset([int(b)])
N = int(one.motion["n_sub"][0])
rr = BlurRenderer(one.faces, one.motion, one.cams, one.H, one.W, one.V, device=dev, cache_visibility=False)
o1 = rr.forward(v, c).cpu().numpy()
print("single-view gpu", o1[0, y, x], "full-batch gpu", out[b, y, x])
for k in range(N):
    ids = torch.full((1, one.H, one.W), -7, dtype=torch.int32, device=dev)
    rr.forward(v, c, ids=ids, ids_subframe=k)
    gid = int(ids[0, y, x].item())
    rk = oracle.render_fwd(one, ids_k=k, eps_amb=1e-6, pixels=[[0, y, x]], sub_range=[[k, k + 1]])
    rs = BlurRenderer(one.faces, one.motion, one.cams, one.H, one.W, one.V, device=dev, sub_range=[[k, k + 1]], cache_visibility=False)
    ok = rs.forward(v, c).cpu().numpy()[0, y, x] * N
    orr = rk["rgba"][0] * N
    d = np.abs(ok - orr).max()
    if d > 1e-3 or gid != rk["ids"][0]:
        print("k %3d gpu id %6d oracle id %6d  gpu %s oracle %s diff %.3g amb_ids %d" % (k, gid, rk["ids"][0], ok, orr, d, rk["amb_ids"][0]))

# geometry of the worst sub-frame's winner
S = oracle.segments(one, 0)
key, valid, Q = oracle.keyframes(one, 0)
sch_s, sch_t = oracle.schedule(N, S, int(one.motion["rule"][0]))
for k in range(N):
    pass
kk = int(os.environ.get("KK", "90"))
ids = torch.full((1, one.H, one.W), -7, dtype=torch.int32, device=dev)
rr.forward(v, c, ids=ids, ids_subframe=kk)
f = int(ids[0, y, x].item())
s, t = int(sch_s[kk]), float(sch_t[kk])
vi = one.faces[f]
P = (1 - t) * key[s][vi] + t * key[s + 1][vi]
W, H = one.W, one.H
pu, pv = -1 + (2 * x + 1) / W, 1 - (2 * y + 1) / H
print("face", f, "verts", vi, "segment", s, "tau", t)
print("corners NDC", P[:, :2].tolist(), "pixel", (pu, pv))
e1, e2 = P[1, :2] - P[0, :2], P[2, :2] - P[0, :2]
area = 0.5 * (e1[0] * e2[1] - e1[1] * e2[0]) * (W / 2) * (H / 2)
print("area px^2 %.4g, edge lengths px" % area, [float(np.linalg.norm((P[(i + 1) % 3, :2] - P[i, :2]) * W / 2)) for i in range(3)])
w, det = oracle.bary_textbook(P[:, 0], P[:, 1], pu, pv)
print("oracle w", w, "colors", one.colors[vi].tolist())
print("keyframes s", key[s][vi].tolist(), "s+1", key[s + 1][vi].tolist())
