"""Diagnostics: stage / list statistics of k4l_raster_fwd on one forward (library built with -DBR_K4L_STATS,
BLURRAST_LIB pointing at it: python tools/build_variants.py stats:BR_K4L_STATS).
usage: BLURRAST_LIB=$PWD/variants/lib_stats.so python tools/k4l_stats.py [C4]"""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import scenes
from paper_2602_07860_b200 import BlurRenderer
sc = scenes.make(sys.argv[1] if len(sys.argv) > 1 else "C4")
dev = torch.device("cuda:0")
r = BlurRenderer(sc.faces, sc.motion, sc.cams, sc.H, sc.W, sc.V, device=dev, cache_visibility=True)
v, c = torch.tensor(sc.verts, device=dev), torch.tensor(sc.colors, device=dev)
r.forward(v, c)
torch.cuda.synchronize()
r.ws[160:256].zero_()
r.forward(v, c)
torch.cuda.synchronize()
st = r.ws[:256].view(torch.int64).cpu().numpy()
names = {20: "pairs (n x ng)", 21: "box-accepted pairs", 22: "staged front", 23: "staged back", 24: "(tau, warp) visits",
         25: "visits with a list", 26: "front list entries", 27: "back entries tested", 28: "back list entries",
         29: "groups"}
for i, nm in names.items():
    print("%-22s %.4e" % (nm, st[i]))
print("faces per visit (front) %.2f, back tested %.2f of %.2f" % (st[26] / st[24], st[27] / st[24], st[28] / st[24]))
