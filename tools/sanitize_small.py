"""Small fwd+bwd runs for compute-sanitizer (C1, a C2 view, a ragged random scene, the fallback path)."""
import sys
import os
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

# soft coverage (K8/K9, grouped, batch and fallback paths), cache off/on, recovery-step kernels
from test_gpu_soft import gpu_soft  # noqa: E402
for sc, kw in [(scenes.make_c1(), {}), (scenes.make_c2().subset([1]), {"sub_range": [[0, 6]]}),
               (scenes.make_c2().subset([3]), {"soft_bin_factor": 1e-9, "sub_range": [[0, 4]]}),
               (scenes.random_mesh_scene(30, 8, H=45, W=61, motion=scenes.rotate((0.2, 1, 0.3), 1.4, N=7, S=3)), {})]:
    G = np.random.default_rng(1).normal(size=(sc.B, sc.H, sc.W, 4)) * 1e-3
    r = gpu_soft(sc, 1e-3, G=G, **kw)
    print("soft", sc.name, "status", r["status"], "alpha", float(r["rgba"][..., 3].sum()), flush=True)
r = gpu_render(scenes.make_c2().subset([0]), G=np.ones((1, 256, 256, 4)) * 1e-4, cache=False)
print("no-cache status", r["status"], flush=True)
import torch  # noqa: E402
from paper_2602_07860_b200 import Recovery  # noqa: E402
tv, f = scenes.icosphere(2, 0.5)
cams = np.stack([scenes.camera_row(scenes.spherical_eye(scenes.CAM_DIST, e, a)) for e, a in [(0, 0), (30, -90)]])
mot = scenes.motion_arrays([scenes.translate((-0.5, 0, 0), N=5)] * 2)
tgt = torch.rand(2, 32, 32, 4, device="cuda")
rec = Recovery(tv.astype(np.float32), f, np.full((len(tv), 3), 0.5, np.float32), cams, mot, tgt, 32, 32, batch=1)
for _ in range(3):
    rec.step()
print("recovery", rec.loss_values(), flush=True)
# the span raster kernels (k_span.cu, BLURRAST_RASTER=span: read per call by the library)
os.environ["BLURRAST_RASTER"] = "span"
for sc in [scenes.make_c1(), scenes.make_c2().subset([1]),
           scenes.random_mesh_scene(40, 5, H=37, W=53, motion=scenes.rotate((0.2, 1, 0.3), 1.2, N=9, S=4))]:
    G = np.random.default_rng(0).normal(size=(sc.B, sc.H, sc.W, 4)) * 1e-3
    r = gpu_render(sc, ids_k=1, G=G)
    print("span", sc.name, "status", r["status"], "sum", float(r["rgba"].sum()), flush=True)
r = gpu_render(scenes.make_c2().subset([2]), ids_k=1, G=np.ones((1, 256, 256, 4)) * 1e-4, bin_factor=1e-9)
print("span fallback status", r["status"], flush=True)
