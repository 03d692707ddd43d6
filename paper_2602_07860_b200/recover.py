"""NEXT-4: translational shape-and-colour recovery from motion-blurred RGBA images (section 5.1,
Eq.16-17; hyper-parameters P:L1469-1474; SPEC S:L402-521 for the loop's interface).

One iteration, all on the device through the C ABI (include/blurrast.h, include/blurrast_optim.h):
  sample a batch of views (seeded shuffle without replacement, reshuffled per epoch)
  -> blur_render_fwd (soft coverage, delta = 1e-4 as the paper; views outside the batch get
     an empty sub-frame range and cost nothing)
  -> blur_l1_loss_grad (Eq.16, mean-reduced over the batch's pixels)
  -> blur_render_bwd (dL_img/dV, dL_img/dC)
  -> blur_laplacian_loss_grad (+ lambda_L dL_L/dV, A21) and blur_smooth_loss_grad (+ lambda_s dL_s/dV, A22)
  -> blur_adam_step on the vertices and on the per-vertex colours (lr 0.01, betas (0.5, 0.99)).
Per-vertex colours stand in for the paper's texture map.  Python only orders the calls.
"""
from __future__ import annotations

import math
from typing import Optional

import numpy as np
import torch

from . import _lib
from .renderer import BlurRenderer


class Recovery:
    def __init__(self, template_verts, faces, template_colors, cams, motion: dict, targets: torch.Tensor, H: int,
                 W: int, delta: float = 1e-4, lambda_s: float = 3e-2, lambda_l: float = 3e-4, lr: float = 0.01,
                 betas=(0.5, 0.99), eps: float = 1e-8, batch: int = 16, seed: int = 0, device="cuda"):
        self.device = torch.device(device)
        self.faces_np = np.ascontiguousarray(np.asarray(faces, np.int32))
        V = int(np.asarray(template_verts).shape[0])
        self.V, self.B = V, int(np.asarray(cams).shape[0])
        self.N = np.asarray(motion["n_sub"], np.int32)
        self.renderer = BlurRenderer(self.faces_np, motion, cams, H, W, V, device=self.device, delta=delta)
        self.verts = torch.tensor(np.asarray(template_verts, np.float32), device=self.device)
        self.verts0 = self.verts.clone()
        self.colors = torch.tensor(np.asarray(template_colors, np.float32), device=self.device)
        self.targets = targets
        self.lambda_s, self.lambda_l = float(lambda_s), float(lambda_l)
        self.lr, self.betas, self.eps = float(lr), (float(betas[0]), float(betas[1])), float(eps)
        self.batch = min(int(batch), self.B)
        self.rng = np.random.default_rng(seed)
        self._queue: list = []
        self.t = 0
        z = lambda x: torch.zeros_like(x)
        self.mv, self.vv, self.mc, self.vc = z(self.verts), z(self.verts), z(self.colors), z(self.colors)
        self.topo = torch.empty(_lib.blur_topology_bytes(V, self.faces_np), dtype=torch.uint8, device=self.device)
        _lib.blur_topology_build(V, self.faces_np, self.topo)
        self.grad = torch.empty_like(targets)
        self.losses = torch.zeros(3, dtype=torch.float32, device=self.device)   # L_img, L_s, L_L
        self.mask = torch.zeros(self.B, dtype=torch.uint8, device=self.device)
        # size the bins on the full view set (every batch needs at most that)
        self.renderer.forward(self.verts, self.colors)

    def next_batch(self):
        if len(self._queue) < self.batch:
            self._queue += list(self.rng.permutation(self.B))
        b, self._queue = self._queue[:self.batch], self._queue[self.batch:]
        return sorted(int(x) for x in b)

    def step(self, views: Optional[list] = None):
        """One iteration; returns the batch of views used.  Asynchronous (no host synchronisation
        except the small batch-mask upload)."""
        views = self.next_batch() if views is None else views
        sub = np.zeros((self.B, 2), np.int32)
        sub[views, 1] = self.N[views]
        self.renderer.set_sub_range(sub)
        m = np.zeros(self.B, np.uint8)
        m[views] = 1
        self.mask.copy_(torch.from_numpy(m))
        r = self.renderer
        out = r.forward(self.verts, self.colors)
        _lib.blur_l1_loss_grad(out, self.targets, self.losses[0:1], self.grad, image_mask=self.mask,
                               n_images=len(views))
        dv, dc = r.backward(self.verts, self.colors, self.grad, reuse_setup=True)
        _lib.blur_laplacian_loss_grad(self.verts, self.verts0, self.topo, self.lambda_l, self.losses[2:3], dv)
        _lib.blur_smooth_loss_grad(self.verts, self.topo, self.lambda_s, self.losses[1:2], dv)
        self.t += 1
        b1, b2 = self.betas
        _lib.blur_adam_step(self.verts, dv, self.mv, self.vv, self.t, self.lr, b1, b2, self.eps)
        _lib.blur_adam_step(self.colors, dc, self.mc, self.vc, self.t, self.lr, b1, b2, self.eps)
        return views

    def loss_values(self) -> dict:
        """L_img, L_s, L_L of the last step and the total of Eq.17 (synchronises)."""
        li, ls, ll = (float(x) for x in self.losses.cpu())
        return dict(img=li, smooth=ls, lap=ll, total=li + self.lambda_s * ls + self.lambda_l * ll)

    def render_all(self) -> torch.Tensor:
        self.renderer.set_sub_range(None)
        return self.renderer.forward(self.verts, self.colors)


def psnr(a: torch.Tensor, b: torch.Tensor) -> float:
    """10 log10(1 / MSE) over all elements, MSE from the blur_sum_sq_diff kernel."""
    out = torch.zeros(1, dtype=torch.float64, device=a.device)
    _lib.blur_sum_sq_diff(a.contiguous(), b.contiguous(), out)
    mse = float(out.item()) / a.numel()
    return math.inf if mse == 0.0 else 10.0 * math.log10(1.0 / mse)


def voxel_iou(va: torch.Tensor, fa: torch.Tensor, vb: torch.Tensor, fb: torch.Tensor, res: int = 32) -> float:
    """3D IoU of two meshes on res^3 voxels, blur_voxel_iou kernel."""
    scratch = torch.empty(_lib.blur_voxel_scratch_bytes(res), dtype=torch.uint8, device=va.device)
    counts = torch.zeros(2, dtype=torch.int64, device=va.device)
    _lib.blur_voxel_iou(va.contiguous(), fa.contiguous(), vb.contiguous(), fb.contiguous(), res, scratch, counts)
    inter, union = (int(x) for x in counts.cpu())
    if union == 0:
        raise ValueError("empty union")
    return inter / union
