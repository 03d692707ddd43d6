"""Diagnostic (GPU, variant build with -DBR_K9_STATS): how K9's work splits between its grouped
(cached-product) path and the per-sub-frame long-bin path on a config.
usage: BLURRAST_LIB=variants/lib_k9stats.so python tools/k9_stats.py [C4] [delta]"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import scenes  # noqa: E402
from paper_2602_07860_b200 import BlurRenderer, _lib  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
delta = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-4
sc = scenes.make(cfg)
dev = torch.device("cuda:0")
r = BlurRenderer(sc.faces, sc.motion, sc.cams, sc.H, sc.W, sc.V, device=dev, delta=delta)
v = torch.tensor(np.asarray(sc.verts, np.float32), device=dev)
c = torch.tensor(np.asarray(sc.colors, np.float32), device=dev)
out = r.forward(v, c)
g = torch.randn_like(out) * 1e-4
lib = _lib.load()
fn = lib.blur_debug_k9_stats
st = (ctypes.c_ulonglong * 8)()
fn(st)
r.backward(v, c, g, reuse_setup=True)
fn(st)
s = list(st)
print(cfg, "grouped groups", s[0], "mean n %.1f" % (s[1] / max(s[0], 1)))
print("pass-2 word items", s[2], "mean faces/word %.1f" % (s[3] / max(s[2], 1)), "mean needing px %.1f" % (s[4] / max(s[2], 1)))
print("long-path sub-frames", s[5], "mean n %.1f" % (s[6] / max(s[5], 1)), "fallback", s[7])
