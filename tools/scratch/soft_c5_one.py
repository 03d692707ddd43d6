"""Scratch: C5 soft (delta 1e-4) fwd + bwd on a subset of views (ncu target for K8/K9)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import scenes
from paper_2602_07860_b200 import BlurRenderer
views = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "0,63").split(",")]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
sc = scenes.make_c5().subset(views)
dev = torch.device("cuda:0")
r = BlurRenderer(sc.faces, sc.motion, sc.cams, sc.H, sc.W, sc.V, device=dev, delta=1e-4, cache_visibility=(os.environ.get("CACHE") == "1") or None)
print("cache flags", r.cache_flags)
v = torch.tensor(np.asarray(sc.verts, np.float32), device=dev)
c = torch.tensor(np.asarray(sc.colors, np.float32), device=dev)
tg = torch.tensor(np.asarray(sc.target, np.float32), device=dev)
for i in range(reps):
    ef = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    eb = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    st = torch.cuda.current_stream()
    ef[0].record(st); out = r.forward(v, c); ef[1].record(st)
    loss, g = r.l2_loss_grad(out, tg)
    eb[0].record(st); r.backward(v, c, g, reuse_setup=True); eb[1].record(st)
    torch.cuda.synchronize()
    print("views %s fwd %.1f ms bwd %.1f ms" % (views, ef[0].elapsed_time(ef[1]), eb[0].elapsed_time(eb[1])), flush=True)
from paper_2602_07860_b200 import _lib
print("hard bins need/cap", _lib.blur_read_bins(r.ws), "soft bins need/cap", _lib.blur_read_soft_bins(r.ws))
try:
    print("status", r.status())
except Exception as e:
    print("status error:", e)
