"""Pins of the oracle's soft background coverage (NEXT-1: Eq.10-15, A17-A20) (-m "not gpu").

Each test names what fixes the expected value: the variational characterisation of a Euclidean
projection onto a convex set, scipy's constrained minimiser, SPEC's worked value (alpha = 0.5 at
squared distance delta ln 2), the exactness of Eq.13 at the keyframes, the delta -> 0 limit
(hard coverage), monotonicity of Eq.15, and central finite differences (exact at the
keyframes by the envelope theorem; exact at any tau where the closest feature is a vertex, since
w^* is then locally constant).
"""
import math

import numpy as np
import pytest
from scipy.optimize import minimize

import oracle
import scenes

rng0 = np.random.default_rng(11)


def _rand_tri(rng):
    while True:
        x, y = rng.uniform(-0.8, 0.8, 3), rng.uniform(-0.8, 0.8, 3)
        det = x[0] * (y[1] - y[2]) - x[1] * (y[0] - y[2]) + x[2] * (y[0] - y[1])
        if abs(det) > 0.05:
            return x, y


def _proj_scipy(x, y, p):
    """Closest point of triangle (x, y) to p by scipy SLSQP over the simplex (library minimiser)."""
    F = np.stack([x, y])
    f = lambda w: float(np.sum((F @ w - p) ** 2))
    g = lambda w: 2.0 * F.T @ (F @ w - p)
    r = minimize(f, np.full(3, 1 / 3), jac=g, method="SLSQP", bounds=[(0, 1)] * 3,
                 constraints=[{"type": "eq", "fun": lambda w: np.sum(w) - 1, "jac": lambda w: np.ones(3)}],
                 options=dict(ftol=1e-15, maxiter=500))
    return r.x, float(np.sum((F @ r.x - p) ** 2))


def test_closest_weights_projection_certificate_and_scipy():
    """A17-A18 closest point vs (i) the projection certificate (q in the triangle and
    (p - q).(v_k - q) <= 0 for every vertex) and (ii) scipy's constrained minimiser."""
    for _ in range(300):
        x, y = _rand_tri(rng0)
        p = rng0.uniform(-1.5, 1.5, 2)
        w, _ = oracle.bary_textbook(x, y, p[0], p[1])
        wh, d2, e, _, _ = oracle.closest_w(x, y, p[0], p[1], w)
        if e < 0:   # inside: w^* = w
            assert np.allclose(wh, w)
            continue
        assert np.all(wh >= 0) and abs(wh.sum() - 1) < 1e-15
        q = np.array([wh @ x, wh @ y])
        assert abs(d2 - np.sum((p - q) ** 2)) < 1e-14
        for k in range(3):
            assert (p - q) @ (np.array([x[k], y[k]]) - q) <= 1e-12
        _, ds = _proj_scipy(x, y, p)
        assert abs(d2 - ds) < 1e-9


def test_closest_weights_inside_returns_w():
    x, y = _rand_tri(rng0)
    w = np.array([0.2, 0.3, 0.5])
    p = np.array([w @ x, w @ y])
    wh, d2, e, _, _ = oracle.closest_w(x, y, p[0], p[1], w)
    assert e == -1 and d2 == 0.0 and np.array_equal(wh, w)


def test_closest_weights_edge_regions():
    """Worked cases on the unit right triangle: edge interior, vertex (t < 0, t > 1)."""
    x, y = np.array([0.0, 1.0, 0.0]), np.array([0.0, 0.0, 1.0])
    wh, d2, e, _, _ = oracle.closest_w(x, y, 0.25, -0.5)      # below edge v0v1: t = 0.25
    assert e == 0 and np.allclose(wh, [0.75, 0.25, 0]) and math.isclose(d2, 0.25)
    wh, d2, _, _, _ = oracle.closest_w(x, y, -1.0, -1.0)       # vertex v0 region
    assert np.allclose(wh, [1, 0, 0]) and math.isclose(d2, 2.0)
    wh, d2, _, _, _ = oracle.closest_w(x, y, 1.0, 1.0)         # hypotenuse midpoint
    assert np.allclose(wh, [0, 0.5, 0.5]) and math.isclose(d2, 0.5)


def test_soft_pair_alpha_half_at_delta_ln2():
    """a pixel at squared distance delta ln 2 outside a lone static triangle has A = 0.5."""
    delta = 1e-4
    X, Y = np.array([-0.5, 0.5, 0.0]), np.array([0.0, 0.0, 0.6])
    r = math.sqrt(delta * math.log(2.0))
    for tau in (0.0, 0.3, 0.5, 0.8, 1.0):
        s = oracle.soft_pair(X, Y, X, Y, tau, 0.1, -r, delta)
        assert abs(s["A"] - 0.5) < 1e-12 and abs(s["d"] - r * r) < 1e-16


def test_soft_pair_exact_at_keyframes_and_upper_bound():
    """Eq.13 is exact when F(tau) = F(X) (tau = 0 or 1): d is the squared distance to the triangle
    (scipy).  At any tau, F(tau) w^* lies in F(tau), so d >= that distance; Eq.12 (exact=True)
    attains it."""
    for _ in range(100):
        X0, Y0 = _rand_tri(rng0)
        X1, Y1 = X0 + rng0.normal(0, 0.2, 3), Y0 + rng0.normal(0, 0.2, 3)
        u, v = rng0.uniform(-1.5, 1.5, 2)
        for tau in (0.0, 1.0, rng0.uniform(0, 1)):
            s = oracle.soft_pair(X0, Y0, X1, Y1, tau, u, v, 1e-2)
            se = oracle.soft_pair(X0, Y0, X1, Y1, tau, u, v, 1e-2, exact=True)
            if s is None:
                continue
            xt, yt = (1 - tau) * X0 + tau * X1, (1 - tau) * Y0 + tau * Y1
            _, dtrue = _proj_scipy(xt, yt, np.array([u, v]))
            assert abs(se["d"] - dtrue) < 1e-9
            assert s["d"] >= dtrue - 1e-9
            if tau in (0.0, 1.0):
                assert abs(s["d"] - dtrue) < 1e-9
            assert math.isclose(s["A"], math.exp(-s["d"] / 1e-2), rel_tol=1e-12)


def test_soft_pair_keyframe_switch_at_half():
    """Eq.13: X = 0 for tau <= 0.5 and X = 1 above; with F(0) = F(1) shifted by a pure translation
    the chosen edge in F(X) differs from the one in F(tau) only through the switch."""
    X0, Y0 = np.array([0.0, 1.0, 0.0]), np.array([0.0, 0.0, 1.0])
    X1, Y1 = X0 + 1.0, Y0.copy()
    # tau = 0.5: F(tau) is shifted by 0.5; p = (0.5 + 0.25, -0.5) has w(tau) = that of (0.25, -0.5)
    s = oracle.soft_pair(X0, Y0, X1, Y1, 0.5, 0.75, -0.5, 1.0)
    assert np.allclose(s["what"], [0.75, 0.25, 0]) and np.allclose(s["pstar"], [0.75, 0.0])
    s2 = oracle.soft_pair(X0, Y0, X1, Y1, 0.5000001, 0.75, -0.5, 1.0)
    assert np.allclose(s2["what"], [0.75, 0.25, 0], atol=1e-6)


def _soft_scene(motion, seed=5, n=6, H=12, W=12):
    return scenes.random_mesh_scene(n, seed, H=H, W=W, motion=motion)


def test_soft_binned_equals_brute_and_pixel_list():
    sc = _soft_scene(scenes.translate((0.5, 0.2, 0.0), N=5))
    a = oracle.render_fwd(sc, mode="brute", delta=2e-3)
    b = oracle.render_fwd(sc, mode="binned", delta=2e-3)
    assert np.array_equal(a["rgba"], b["rgba"])
    pix = np.array([[0, j, i] for j in range(0, 12, 3) for i in range(12)])
    c = oracle.render_fwd(sc, delta=2e-3, pixels=pix)
    assert np.array_equal(c["rgba"], b["rgba"][0][pix[:, 1], pix[:, 2]])


def test_soft_alpha_range_rgb_unchanged_and_delta_limit():
    """RGB is untouched by the background term (background colour 0, aggregate function off,
    P:L1180); alpha in [0, 1]; alpha -> hard coverage as delta -> 0."""
    sc = _soft_scene(scenes.rotate((0.1, 1, 0.2), 1.2, N=6, S=2))
    h = oracle.render_fwd(sc)
    s = oracle.render_fwd(sc, delta=1e-2)
    assert np.array_equal(h["rgba"][..., :3], s["rgba"][..., :3])
    assert s["rgba"][..., 3].min() >= 0 and s["rgba"][..., 3].max() <= 1
    assert np.all(s["rgba"][..., 3] >= h["rgba"][..., 3])
    assert (s["rgba"][..., 3] > h["rgba"][..., 3] + 1e-3).sum() > 10
    z = oracle.render_fwd(sc, delta=1e-14)
    assert np.max(np.abs(z["rgba"] - h["rgba"])) < 1e-12


def test_soft_alpha_monotone_in_faces_and_delta():
    """Eq.15 is monotone in every A_j: removing a face never raises alpha; A = exp(-d/delta)
    grows with delta."""
    sc = _soft_scene(scenes.translate((0.4, -0.2, 0.1), N=4), n=7)
    full = oracle.render_fwd(sc, delta=5e-3)["rgba"][..., 3]
    import dataclasses
    for drop in range(sc.F):
        keep = np.array([f for f in range(sc.F) if f != drop])
        sub = dataclasses.replace(sc, faces=sc.faces[keep])
        assert np.all(oracle.render_fwd(sub, delta=5e-3)["rgba"][..., 3] <= full + 1e-15)
    big = oracle.render_fwd(sc, delta=2e-2)["rgba"][..., 3]
    assert np.all(big >= full - 1e-15)


def test_soft_single_static_triangle_closed_form():
    """One static triangle: background alpha = exp(-dist^2 / delta) with dist the Euclidean
    distance of the pixel centre to the projected triangle (scipy), Eq.10 with one face."""
    verts = np.array([[-0.6, -0.4, 0.0], [0.5, -0.5, 0.0], [0.1, 0.6, 0.0]])
    sc = scenes.single_scene(verts, [[0, 1, 2]], np.ones((3, 3)) * 0.5, H=10, W=10)
    delta = 3e-2
    r = oracle.render_fwd(sc, delta=delta)
    key, _, _ = oracle.keyframes(sc)
    x, y = key[0, :, 0], key[0, :, 1]
    for j in range(10):
        for i in range(10):
            if r["ids"][0, j, i] >= 0 or r["rgba"][0, j, i, 3] == 1.0:
                continue
            p = np.array([-1 + (2 * i + 1) / 10, 1 - (2 * j + 1) / 10])
            _, d = _proj_scipy(x, y, p)
            assert abs(r["rgba"][0, j, i, 3] - math.exp(-d / delta)) < 1e-8


def _winners(sc):
    N = int(sc.motion["n_sub"][0])
    fz = np.zeros((N, sc.H, sc.W), np.int32)
    for k in range(N):
        fz[k] = oracle.render_fwd(sc, ids_k=k)["ids"][0]
    return fz.reshape(-1)


def _fd_verts(sc, G, fz, delta, h=1e-6):
    V64 = sc.verts.astype(np.float64)
    num = np.zeros((sc.V, 3))
    for v in range(sc.V):
        for c in range(3):
            vp, vm = V64.copy(), V64.copy()
            vp[v, c] += h
            vm[v, c] -= h
            lp = np.sum(G * oracle.render_fwd(sc, frozen=fz, verts=vp, delta=delta)["rgba"])
            lm = np.sum(G * oracle.render_fwd(sc, frozen=fz, verts=vm, delta=delta)["rgba"])
            num[v, c] = (lp - lm) / (2 * h)
    return num


@pytest.mark.parametrize("motion", [scenes.translate((0.6, 0.2, -0.3), N=2),
                                    scenes.rotate((0.2, 1, 0.1), 1.2, N=4, S=3)])
def test_soft_backward_fd_at_keyframes(motion):
    """Sub-frames at tau in {0, 1} only (N = 2, S = 1; N = S + 1): Eq.13 is exact there and, by the
    envelope theorem, the derivative with w^* frozen equals the derivative of the distance itself,
    so frozen-coverage central differences of the full forward pin the soft backward (alpha
    channel), including the keyframe split, projection, camera and pose chain."""
    sc = _soft_scene(motion, seed=9, n=6)
    delta = 1e-2
    rng = np.random.default_rng(3)
    G = rng.normal(size=(1, sc.H, sc.W, 4))
    fz = _winners(sc)
    dv, _ = oracle.render_bwd(sc, G, delta=delta)
    dv_hard, _ = oracle.render_bwd(sc, G)
    num = _fd_verts(sc, G, fz, delta)
    assert np.linalg.norm(dv - num) / np.linalg.norm(num) < 1e-6
    assert np.linalg.norm(dv - dv_hard) > 1e-3 * np.linalg.norm(dv)   # the soft term is really there


def test_soft_backward_fd_vertex_regions_generic_tau():
    """Generic tau (N = 4: tau = 1/3, 2/3 use F(0) / F(1) as F(X)): where a pixel's closest feature
    on its face's F(X) is a vertex, w^* is locally constant and the frozen-w^* derivative is the
    true one; with the loss restricted to such pixels, central differences pin the generic-tau
    backward (including the (1 - tau, tau) split onto keyframes)."""
    verts = np.array([[-0.5, -0.3, 0.2], [0.4, -0.45, -0.1], [0.05, 0.5, 0.0]])
    sc = scenes.single_scene(verts, [[0, 1, 2]], np.ones((3, 3)) * 0.5, H=14, W=14,
                             motion=scenes.translate((0.5, 0.3, 0.0), N=4))
    delta = 2e-2
    key, _, _ = oracle.keyframes(sc)
    _, taus = oracle.schedule(4, 1)
    G = np.zeros((1, 14, 14, 4))
    n_sel = 0
    for j in range(14):
        for i in range(14):
            u, v = -1 + (2 * i + 1) / 14, 1 - (2 * j + 1) / 14
            ok = True
            for t in taus:
                s = oracle.soft_pair(key[0, :, 0], key[0, :, 1], key[1, :, 0], key[1, :, 1], t, u, v, delta)
                w, _ = oracle.bary_textbook((1 - t) * key[0, :, 0] + t * key[1, :, 0],
                                            (1 - t) * key[0, :, 1] + t * key[1, :, 1], u, v)
                if w is not None and np.all(w >= 0):
                    continue       # covered at this sub-frame: alpha 1, no gradient
                if s is None or np.max(s["what"]) < 1.0 or s["A"] < 1e-6:
                    ok = False
            if ok:
                G[0, j, i, 3] = 1.0 + 0.1 * i - 0.05 * j
                n_sel += 1
    assert n_sel > 5
    fz = _winners(sc)
    dv, _ = oracle.render_bwd(sc, G, delta=delta)
    num = _fd_verts(sc, G, fz, delta)
    assert np.linalg.norm(num) > 1e-3
    assert np.linalg.norm(dv - num) / np.linalg.norm(num) < 1e-6


def test_soft_backward_pixel_list_and_linearity():
    sc = _soft_scene(scenes.translate((0.5, 0.1, 0.0), N=3), seed=21)
    rng = np.random.default_rng(4)
    G1, G2 = rng.normal(size=(2, 1, sc.H, sc.W, 4))
    a, _ = oracle.render_bwd(sc, G1, delta=1e-2)
    b, _ = oracle.render_bwd(sc, G2, delta=1e-2)
    c, _ = oracle.render_bwd(sc, 2 * G1 - G2, delta=1e-2)
    assert np.allclose(c, 2 * a - b, rtol=1e-10, atol=1e-12)
    pix = np.array([[0, j, i] for j in range(sc.H) for i in range(sc.W)])
    d, _ = oracle.render_bwd(sc, G1.reshape(-1, 4), delta=1e-2, pixels=pix)
    assert np.allclose(d, a, rtol=1e-10, atol=1e-12)
