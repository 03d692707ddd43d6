"""Pins of the NEXT-4 oracle (oracle/optim.py) against closed forms, invariances, finite differences
and hand-traced recurrences (-m "not gpu"): SPEC S:L424-490 examples and invariants."""
import math

import numpy as np
import pytest

import scenes
from oracle import optim

rng0 = np.random.default_rng(13)


def test_l1_loss_closed_forms_and_fd():
    a = rng0.uniform(0, 1, (3, 5, 4, 4))
    assert optim.l1_image_loss(a, a)[0] == 0.0
    b = a.copy()
    b[..., 3] += 0.1                      # rendered = target + 0.1 on alpha only -> 0.1
    assert abs(optim.l1_image_loss(b, a)[0] - 0.1) < 1e-12
    t = rng0.uniform(0, 1, a.shape)
    loss, g = optim.l1_image_loss(a, t)
    h = 1e-6
    for _ in range(20):
        idx = tuple(rng0.integers(0, s) for s in a.shape)
        ap, am = a.copy(), a.copy()
        ap[idx] += h
        am[idx] -= h
        num = (optim.l1_image_loss(ap, t)[0] - optim.l1_image_loss(am, t)[0]) / (2 * h)
        assert abs(num - g[idx]) < 1e-8
    # image mask: only the batch's images count, and they are normalised by their own pixel count
    m = np.array([True, False, True])
    lm, gm = optim.l1_image_loss(a, t, m)
    l2, _ = optim.l1_image_loss(a[m], t[m])
    assert abs(lm - l2) < 1e-15 and np.all(gm[1] == 0)


def test_laplacian_closed_forms():
    v, f = scenes.star(6)
    assert optim.laplacian_loss(v, v, f)[0] == 0.0
    shift = v + np.array([0.3, -0.2, 0.7])          # global translation -> 0
    assert optim.laplacian_loss(shift, v, f)[0] < 1e-28
    d = np.array([0.1, 0.2, -0.3])
    w = v.copy()
    w[0] += d                                       # centre displaced on a symmetric star
    # centre: r = d; ring vertex: neighbours (centre + 2 ring) -> r = -d/3
    expect = float(d @ d) * (1.0 + 6.0 / 9.0)
    assert abs(optim.laplacian_loss(w, v, f)[0] - expect) < 1e-14


def test_laplacian_gradient_fd_and_translation_invariance():
    v, f = scenes.icosphere(1, 1.0)
    x = v + rng0.normal(0, 0.05, v.shape)
    L, g = optim.laplacian_loss(x, v, f)
    h = 1e-6
    for i in rng0.choice(len(v), 6, replace=False):
        for c in range(3):
            xp, xm = x.copy(), x.copy()
            xp[i, c] += h
            xm[i, c] -= h
            num = (optim.laplacian_loss(xp, v, f)[0] - optim.laplacian_loss(xm, v, f)[0]) / (2 * h)
            assert abs(num - g[i, c]) < 1e-7
    assert abs(g.sum(0)).max() < 1e-12                # translation invariance: gradient sums to 0
    assert abs(optim.laplacian_loss(x + 0.5, v + 0.5, f)[0] - L) < 1e-12


def test_smoothness_closed_forms():
    # two coplanar faces, consistent orientation: theta = pi -> 0
    v = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [1, -1, 0.0]])
    f = np.array([[0, 1, 2], [1, 0, 3]])
    assert abs(optim.smooth_loss(v, f)[0]) < 1e-28
    # folded flat: the two wings coincide, theta = 0 -> (1 + 1)^2 = 4
    v2 = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0.5, 1, 0.0]])
    assert abs(optim.smooth_loss(v2, f)[0] - 4.0) < 1e-12
    # right dihedral angle: cos = 0 -> 1
    v3 = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0.3, 0, 1.0]])
    assert abs(optim.smooth_loss(v3, f)[0] - 1.0) < 1e-12


def test_smoothness_fd_and_rigid_invariance():
    v, f = scenes.icosphere(1, 1.0)
    x = v + rng0.normal(0, 0.05, v.shape)
    L, g = optim.smooth_loss(x, f)
    assert len(optim.interior_edges(f)) == 120          # closed icosphere-1: every edge interior
    h = 1e-6
    for i in rng0.choice(len(v), 6, replace=False):
        for c in range(3):
            xp, xm = x.copy(), x.copy()
            xp[i, c] += h
            xm[i, c] -= h
            num = (optim.smooth_loss(xp, f)[0] - optim.smooth_loss(xm, f)[0]) / (2 * h)
            assert abs(num - g[i, c]) < 1e-6 * max(1.0, abs(num))
    from scipy.spatial.transform import Rotation
    R = Rotation.from_rotvec([0.3, -0.5, 0.9]).as_matrix()
    assert abs(optim.smooth_loss(2.0 * x @ R.T + 1.5, f)[0] - L) < 1e-10   # similarity invariance


def test_adam_hand_traces():
    p, g = np.array([0.7]), np.array([0.0])
    z = np.zeros(1)
    q, m, v = optim.adam_step(p, g, z, z, 1)
    assert np.array_equal(q, p)                          # zero gradient -> unchanged
    lr, b1, b2, eps = 0.01, 0.5, 0.99, 1e-8
    g = np.array([0.3])
    q1, m1, v1 = optim.adam_step(p, g, z, z, 1, lr, b1, b2, eps)
    assert abs(q1[0] - (0.7 - lr * 0.3 / (0.3 + eps))) < 1e-15        # m^ = g, v^ = g^2
    q2, m2, v2 = optim.adam_step(q1, g, m1, v1, 2, lr, b1, b2, eps)
    # constant gradient: m2 = (1 - b1)(1 + b1) g, v2 = (1 - b2)(1 + b2) g^2 -> again m^ = g, v^ = g^2
    assert abs(m2[0] - (1 - b1) * (1 + b1) * 0.3) < 1e-16 and abs(v2[0] - (1 - b2) * (1 + b2) * 0.09) < 1e-16
    assert abs(q2[0] - (q1[0] - lr * 0.3 / (0.3 + eps))) < 1e-15


def test_voxel_iou_closed_forms():
    v, f = scenes.cube(0.5)
    assert optim.voxel_iou(v, f, v, f, 16) == 1.0
    v2, f2 = scenes.cube(0.5, centre=(3.0, 0, 0))
    assert optim.voxel_iou(v, f, v2, f2, 16) == 0.0
    # cube vs the same cube scaled 0.5 about its centre -> 1/8 (within 0.02 at 32^3)
    assert abs(optim.voxel_iou(v, f, 0.5 * v, f, 32) - 0.125) < 0.02
    # a sphere (icosphere-3) vs itself and vs a half-size copy: volume ratio 1/8 within 0.03
    s, fs = scenes.icosphere(3, 1.0)
    assert abs(optim.voxel_iou(s, fs, 0.5 * s, fs, 32) - 0.125) < 0.03


def test_psnr_closed_forms():
    a = rng0.uniform(0, 1, (4, 4, 3))
    assert optim.psnr(a, a) == math.inf
    assert abs(optim.psnr(a, a + 0.1) - 20.0) < 1e-9
    b = rng0.uniform(0, 1, a.shape)
    assert abs(optim.psnr(a, b) - 10 * math.log10(1 / np.mean((a - b) ** 2))) < 1e-12
