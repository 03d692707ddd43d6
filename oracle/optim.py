"""fp64 CPU oracle of the NEXT-4 translational inverse-rendering step (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may import this module.  It
shares no code with the CUDA path.  Every function follows the passage it cites; gradients of the
regularisers come from torch autograd in fp64 on the plainly written loss (a library primitive used
as a step), everything else is written out.  Pins: tests/test_oracle_optim.py.

  l1_image_loss   Eq.16: L_img = ||I - I^||_1 + ||alpha - alpha^||_1, each mean-reduced
                  over its channels (reading Q22), adjoint sign(I^ - I) / n, sign(0) = 0.
  laplacian_loss  A21: sum_v || delta_v - mean_{v' in N(v)} delta_v' ||^2,
                  delta = V - V_template, N(v) = vertices sharing an edge with v.
  smooth_loss     A22: sum over edges shared by exactly two faces of (cos theta + 1)^2,
                  theta the dihedral angle between the faces (pi when flat; edges of a degenerate
                  face skipped).
  total_loss      Eq.17: L_img + lambda_s L_s + lambda_L L_L.
  adam_step       Adam (alpha = 0.01, beta = (0.5, 0.99)), bias-corrected, eps = 1e-8.
  voxel_iou       3D IoU on res^3 voxels: occupancy of voxel centres by parity of
                  the +x ray's face crossings, on the shared bounding cube of both meshes.
  psnr            10 log10(1 / MSE).
"""
from __future__ import annotations

import math

import numpy as np


def l1_image_loss(out, target, images=None):
    """(loss, grad [B,H,W,4]).  images: optional bool [B] mask of the images in the batch."""
    out = np.asarray(out, np.float64)
    target = np.asarray(target, np.float64)
    B = out.shape[0]
    mask = np.ones(B, bool) if images is None else np.asarray(images, bool)
    npx = int(mask.sum()) * out.shape[1] * out.shape[2]
    diff = out - target
    grad = np.zeros_like(out)
    if npx == 0:
        return 0.0, grad
    d = diff[mask]
    loss = np.abs(d[..., :3]).sum() / (3.0 * npx) + np.abs(d[..., 3]).sum() / npx
    g = np.sign(d)
    g[..., :3] /= 3.0 * npx
    g[..., 3] /= npx
    grad[mask] = g
    return float(loss), grad


def neighbours(faces, V):
    """N(v): the vertices sharing an edge with v (sorted lists)."""
    nb = [set() for _ in range(V)]
    for f in np.asarray(faces):
        for i in range(3):
            a, b = int(f[i]), int(f[(i + 1) % 3])
            if a != b:
                nb[a].add(b)
                nb[b].add(a)
    return [sorted(s) for s in nb]


def _torch():
    import torch
    return torch


def laplacian_loss(verts, verts0, faces):
    """(loss, dL/dverts [V,3]) of A21 for the displacement delta = verts - verts0."""
    torch = _torch()
    V = len(verts)
    nb = neighbours(faces, V)
    x = torch.tensor(np.asarray(verts, np.float64), requires_grad=True)
    delta = x - torch.tensor(np.asarray(verts0, np.float64))
    loss = torch.zeros((), dtype=torch.float64)
    for v in range(V):
        if not nb[v]:
            continue            # isolated vertex: no term
        mean = sum(delta[u] for u in nb[v]) / len(nb[v])
        r = delta[v] - mean
        loss = loss + (r * r).sum()
    loss.backward()
    return float(loss.detach()), x.grad.numpy().copy()


def interior_edges(faces):
    """Edges shared by exactly two faces: list of (a, b, c, d), c and d the opposite vertices."""
    m = {}
    for fi, f in enumerate(np.asarray(faces)):
        for i in range(3):
            a, b, c = int(f[i]), int(f[(i + 1) % 3]), int(f[(i + 2) % 3])
            key = (min(a, b), max(a, b))
            m.setdefault(key, []).append(c)
    return [(k[0], k[1], cs[0], cs[1]) for k, cs in sorted(m.items()) if len(cs) == 2]


def _cos_dihedral(torch, pa, pb, pc, pd):
    """cos of the dihedral angle at edge ab between faces (a, b, c) and (a, b, d): the angle between
    the components of c - a and d - a perpendicular to the edge (pi for a flat pair)."""
    e = pb - pa
    ee = (e * e).sum()
    u = (pc - pa) - ((pc - pa) * e).sum() / ee * e
    w = (pd - pa) - ((pd - pa) * e).sum() / ee * e
    return (u * w).sum() / torch.sqrt((u * u).sum() * (w * w).sum())


def smooth_loss(verts, faces):
    """(loss, dL/dverts [V,3]) of A22."""
    torch = _torch()
    x = torch.tensor(np.asarray(verts, np.float64), requires_grad=True)
    loss = torch.zeros((), dtype=torch.float64)
    for a, b, c, d in interior_edges(faces):
        pa, pb, pc, pd = x[a], x[b], x[c], x[d]
        e = pb - pa
        if float((e * e).sum().detach()) == 0.0:
            continue
        ee = (e * e).sum()
        u = (pc - pa) - ((pc - pa) * e).sum() / ee * e
        w = (pd - pa) - ((pd - pa) * e).sum() / ee * e
        if float((u * u).sum().detach()) == 0.0 or float((w * w).sum().detach()) == 0.0:
            continue                # degenerate face: edge skipped
        cs = _cos_dihedral(torch, pa, pb, pc, pd)
        loss = loss + (cs + 1.0) ** 2
    if loss.requires_grad:
        loss.backward()
        g = x.grad.numpy().copy()
    else:
        g = np.zeros_like(np.asarray(verts, np.float64))
    return float(loss.detach()), g


def adam_step(p, g, m, v, t, lr=0.01, b1=0.5, b2=0.99, eps=1e-8):
    """One Adam step at (1-based) step t; returns (p, m, v) new arrays (fp64)."""
    p, g, m, v = (np.asarray(a, np.float64) for a in (p, g, m, v))
    m = b1 * m + (1.0 - b1) * g
    v = b2 * v + (1.0 - b2) * g * g
    mh = m / (1.0 - b1 ** t)
    vh = v / (1.0 - b2 ** t)
    return p - lr * mh / (np.sqrt(vh) + eps), m, v


def _occupancy(verts, faces, lo, size, res):
    """Voxel-centre occupancy by the parity of +x ray crossings.  The ray origin is nudged by
    (1e-7 sqrt2, 1e-7 sqrt3) voxel in (y, z) so that it never passes exactly through an edge."""
    verts = np.asarray(verts, np.float64)
    faces = np.asarray(faces)
    h = size / res
    occ = np.zeros((res, res, res), bool)
    ny, nz = 1e-7 * math.sqrt(2.0) * h, 1e-7 * math.sqrt(3.0) * h
    tri = verts[faces]                                     # [F,3,3]
    for j in range(res):
        y = lo[1] + (j + 0.5) * h + ny
        for k in range(res):
            z = lo[2] + (k + 0.5) * h + nz
            # faces whose (y, z) projection contains (y, z): signed areas of the sub-triangles
            y0, z0 = tri[:, 0, 1], tri[:, 0, 2]
            y1, z1 = tri[:, 1, 1], tri[:, 1, 2]
            y2, z2 = tri[:, 2, 1], tri[:, 2, 2]
            s0 = (y1 - y) * (z2 - z) - (y2 - y) * (z1 - z)
            s1 = (y2 - y) * (z0 - z) - (y0 - y) * (z2 - z)
            s2 = (y0 - y) * (z1 - z) - (y1 - y) * (z0 - z)
            inside = ((s0 > 0) & (s1 > 0) & (s2 > 0)) | ((s0 < 0) & (s1 < 0) & (s2 < 0))
            if not inside.any():
                continue
            den = s0 + s1 + s2
            xhit = (s0 * tri[:, 0, 0] + s1 * tri[:, 1, 0] + s2 * tri[:, 2, 0]) / np.where(inside, den, 1.0)
            xs = np.sort(xhit[inside])
            for i in range(res):
                x = lo[0] + (i + 0.5) * h
                occ[i, j, k] = (np.count_nonzero(xs > x) % 2) == 1
    return occ


def bounding_cube(va, vb):
    """Shared bounding cube of two vertex sets: (lower corner, edge length), 1% margin."""
    pts = np.concatenate([np.asarray(va, np.float64), np.asarray(vb, np.float64)])
    lo, hi = pts.min(0), pts.max(0)
    c = 0.5 * (lo + hi)
    size = float((hi - lo).max()) * 1.02
    return c - 0.5 * size, size


def voxel_iou(va, fa, vb, fb, res=32):
    lo, size = bounding_cube(va, vb)
    a = _occupancy(va, fa, lo, size, res)
    b = _occupancy(vb, fb, lo, size, res)
    union = np.count_nonzero(a | b)
    if union == 0:
        raise ValueError("empty union")
    return np.count_nonzero(a & b) / union


def psnr(a, b):
    mse = float(np.mean((np.asarray(a, np.float64) - np.asarray(b, np.float64)) ** 2))
    return math.inf if mse == 0.0 else 10.0 * math.log10(1.0 / mse)
