"""Scratch: front/back list statistics of k4l_raster_fwd (build with -DBR_K4L_STATS) on one C4 forward."""
import os, sys, ctypes
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import scenes
from paper_2602_07860_b200 import BlurRenderer
sc = scenes.make(sys.argv[1] if len(sys.argv) > 1 else "C4")
dev = torch.device("cuda:0")
r = BlurRenderer(sc.faces, sc.motion, sc.cams, sc.H, sc.W, sc.V, device=dev, cache_visibility=False)
v, c = torch.tensor(sc.verts, device=dev), torch.tensor(sc.colors, device=dev)
r.forward(v, c)
torch.cuda.synchronize()
ws = r.ws
st = ws[:256].view(torch.int32).cpu().numpy()
print("front iters", st[40], "back iters", st[41], "back culled", st[42], "warp-tau with zmax finite", st[43], "of", st[44])
print("orient", ws[64:72].view(torch.float64).item())
