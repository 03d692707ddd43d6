"""Kernel timings of the raster fwd/bwd on a config with the visibility cache on/off (diagnostics).
usage: python tools/time_raster.py [C4] [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import scenes
from paper_2602_07860_b200 import BlurRenderer
cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
sc = scenes.make(cfg)
dev = torch.device("cuda:0")
v, c = torch.tensor(sc.verts, device=dev), torch.tensor(sc.colors, device=dev)
st = torch.cuda.current_stream()
for cache in (True, False):
    r = BlurRenderer(sc.faces, sc.motion, sc.cams, sc.H, sc.W, sc.V, device=dev, cache_visibility=cache)
    out = r.forward(v, c)
    g = torch.randn_like(out) * 1e-6
    fw, bw = [], []
    for i in range(reps + 2):
        ef = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        eb = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        for e in ef + eb:
            e.record(st)          # the C ABI re-records them around the raster kernels
        r.forward(v, c, out=out, events=ef)
        r.backward(v, c, g, reuse_setup=True, events=eb)
        torch.cuda.synchronize()
        if i >= 2:
            fw.append(ef[0].elapsed_time(ef[1])); bw.append(eb[0].elapsed_time(eb[1]))
    print("%s %s cache=%d fwd %.3f ms bwd %.3f ms" % (os.environ.get("BLURRAST_RASTER", "legacy"), cfg, cache, np.median(fw), np.median(bw)), flush=True)
    del r
