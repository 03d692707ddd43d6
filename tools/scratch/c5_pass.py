"""Scratch: one C5 pass (2 images, cache on) fwd + bwd, for a launch list."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import scenes
from paper_2602_07860_b200 import BlurRenderer
sc = scenes.make_c5().subset([0, 63])
dev = torch.device("cuda:0")
r = BlurRenderer(sc.faces, sc.motion, sc.cams, sc.H, sc.W, sc.V, device=dev)
v = torch.tensor(np.asarray(sc.verts, np.float32), device=dev)
c = torch.tensor(np.asarray(sc.colors, np.float32), device=dev)
for i in range(3):
    out = r.forward(v, c)
    r.backward(v, c, torch.randn_like(out) * 1e-6, reuse_setup=True)
torch.cuda.synchronize()
print("cache flags", r.cache_flags)
