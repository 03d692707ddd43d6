"""Census of the span raster's forward on a config (diagnostics): covered pairs, shades, tests, records,
grouped-path groups / pairs / sub-frames.  usage: BLURRAST_RASTER=span python tools/census_span.py [C4]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import scenes
from paper_2602_07860_b200 import BlurRenderer
cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
sc = scenes.make(cfg)
dev = torch.device("cuda:0")
r = BlurRenderer(sc.faces, sc.motion, sc.cams, sc.H, sc.W, sc.V, device=dev)
v, c = torch.tensor(sc.verts, device=dev), torch.tensor(sc.colors, device=dev)
r.forward(v, c)
cen = torch.zeros(12, dtype=torch.int64, device=dev)
r.forward(v, c, census=cen)
x = cen.cpu().numpy().astype(float)
T = (sc.H // 16) * (sc.W // 16)
print(cfg, "frag %.3g shade %.3g tests %.3g records %.3g | groups %.3g pairs %.3g subframes %.3g | pairs/group %.1f ng %.2f n %.1f recs/group %.1f frag/rec %.2f"
      % (x[0], x[1], x[2], x[3], x[5], x[6], x[7], x[6] / max(x[5], 1), x[7] / max(x[5], 1), x[6] / max(x[7], 1), x[3] / max(x[5], 1), x[0] / max(x[3], 1)))
