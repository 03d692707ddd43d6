"""Small fwd+bwd runs for compute-sanitizer (C1, a C2 view, a ragged random scene, the fallback path)."""
import sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
import scenes
from test_gpu_parity import gpu_render

for sc, kw in [(scenes.make_c1(), {}), (scenes.make_c2().subset([1]), {}),
               (scenes.make_c2().subset([2]), {"bin_factor": 1e-9}),
               (scenes.random_mesh_scene(40, 5, H=37, W=53, motion=scenes.rotate((0.2, 1, 0.3), 1.2, N=9, S=4)), {})]:
    G = np.random.default_rng(0).normal(size=(sc.B, sc.H, sc.W, 4)) * 1e-3
    r = gpu_render(sc, ids_k=1, G=G, **kw)
    print(sc.name, sc.H, sc.W, "status", r["status"], "sum", float(r["rgba"].sum()), flush=True)
