"""Property-based pins of the oracle (hypothesis, -m "not gpu"): invariants the paper fixes, checked on
random small inputs rather than hand-picked ones.

  * the fast solver (Eq.8 with the literal A11-A16 coefficients) equals the textbook solve of the
    lerped triangle at any t (Eq.5-8 are exact under linear motion), and its weights sum to 1;
  * barycentric weights are non-negative exactly inside and reproduce the point;
  * the brute and binned oracle modes are bit-identical (the bbox cull is exact);
  * the blurred image is the mean of its sub-frame ranges, and alpha is in [0, 1];
  * the closest-point weights (A17-A18) are a convex combination on the triangle's boundary whose
    distance is never larger than any vertex's or any edge midpoint's.
"""
import numpy as np
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

import oracle
import scenes

coord = st.floats(-0.9, 0.9, allow_nan=False, width=64)
SETTINGS = dict(max_examples=60, deadline=None, derandomize=True, suppress_health_check=[HealthCheck.too_slow])


def _tri(xs):
    x, y = np.array(xs[:3]), np.array(xs[3:6])
    det = x[0] * (y[1] - y[2]) - x[1] * (y[0] - y[2]) + x[2] * (y[0] - y[1])
    return x, y, det


@settings(**SETTINGS)
@given(st.lists(coord, min_size=12, max_size=12), st.floats(0, 1), coord, coord)
def test_fast_solver_equals_textbook_at_any_t(xs, t, u, v):
    X0, Y0, _ = _tri(xs[:6])
    X1, Y1, _ = _tri(xs[6:])
    Xt, Yt = (1 - t) * X0 + t * X1, (1 - t) * Y0 + t * Y1
    wt, det = oracle.bary_textbook(Xt, Yt, u, v)
    if wt is None or abs(det) < 1e-3:
        return
    wf, den = oracle.fast_eval(X0, Y0, X1, Y1, u, v, t)
    assert wf is not None
    assert np.allclose(wf, wt, rtol=1e-8, atol=1e-8 * max(1.0, np.abs(wt).max()))
    assert abs(wf.sum() - 1.0) < 1e-9 * max(1.0, np.abs(wf).max())


@settings(**SETTINGS)
@given(st.lists(coord, min_size=6, max_size=6), st.lists(st.floats(0, 1), min_size=3, max_size=3))
def test_weights_reproduce_point_and_sign_means_inside(xs, lam):
    x, y, det = _tri(xs)
    if abs(det) < 1e-3:
        return
    lam = np.array(lam) + 1e-3
    lam /= lam.sum()
    u, v = lam @ x, lam @ y                       # a point strictly inside
    w, _ = oracle.bary_textbook(x, y, u, v)
    assert np.all(w >= -1e-12) and np.allclose(w, lam, atol=1e-9)
    u2, v2 = x[0] + 1.5 * (x[0] - lam @ x), y[0] + 1.5 * (y[0] - lam @ y)   # beyond vertex 0: outside
    w2, _ = oracle.bary_textbook(x, y, u2, v2)
    assert w2.min() < 0 and abs(w2 @ x - u2) < 1e-9 and abs(w2 @ y - v2) < 1e-9


@settings(max_examples=12, deadline=None, derandomize=True, suppress_health_check=[HealthCheck.too_slow])
@given(st.integers(0, 10_000), st.sampled_from(["translate", "rotate"]))
def test_brute_equals_binned_and_sub_ranges_add_up(seed, kind):
    motion = scenes.translate((0.5, 0.2, -0.3), N=5) if kind == "translate" else scenes.rotate((0.3, 1, 0.1), 1.1, N=6, S=2)
    sc = scenes.random_mesh_scene(6, seed, H=10, W=12, motion=motion)
    a = oracle.render_fwd(sc, mode="brute")["rgba"]
    b = oracle.render_fwd(sc, mode="binned")["rgba"]
    assert np.array_equal(a, b)
    N = int(sc.motion["n_sub"][0])
    k = N // 2
    p = oracle.render_fwd(sc, sub_range=[[0, k]])["rgba"] + oracle.render_fwd(sc, sub_range=[[k, N]])["rgba"]
    assert np.allclose(p, a, atol=1e-14)
    assert a[..., 3].min() >= 0 and a[..., 3].max() <= 1 + 1e-15
    s = oracle.render_fwd(sc, delta=5e-3)["rgba"]
    assert s[..., 3].min() >= 0 and s[..., 3].max() <= 1 + 1e-15


@settings(**SETTINGS)
@given(st.lists(coord, min_size=6, max_size=6), st.floats(-2, 2), st.floats(-2, 2))
def test_closest_weights_are_convex_and_no_farther_than_vertices_or_midpoints(xs, pu, pv):
    x, y, det = _tri(xs)
    if abs(det) < 1e-3:
        return
    w, _ = oracle.bary_textbook(x, y, pu, pv)
    wh, d2, e, _, _ = oracle.closest_w(x, y, pu, pv, w)
    assert np.all(wh >= 0) and abs(wh.sum() - 1) < 1e-12
    if e >= 0:
        assert np.min(wh) == 0.0                    # on the boundary: some weight is exactly 0
    p = np.array([pu, pv])
    cands = [np.array([x[i], y[i]]) for i in range(3)]
    cands += [0.5 * (cands[i] + cands[(i + 1) % 3]) for i in range(3)]
    assert all(d2 <= np.sum((p - c) ** 2) + 1e-12 for c in cands)


def _seg_dist2(px, py, ax, ay, bx, by):
    """Squared distance from a point to a segment (textbook clamp of the projection)."""
    dx, dy = bx - ax, by - ay
    L = dx * dx + dy * dy
    t = 0.0 if L == 0 else min(1.0, max(0.0, ((px - ax) * dx + (py - ay) * dy) / L))
    qx, qy = ax + t * dx - px, ay + t * dy - py
    return qx * qx + qy * qy


@settings(**SETTINGS)
@given(st.lists(coord, min_size=12, max_size=12), st.floats(0, 1), st.floats(-2, 2), st.floats(-2, 2))
def test_soft_distance_bounds_true_distance(xs, tau, u, v):
    """Eq.14's d = |p - F(tau) w*|^2 with w* convex (A17-A18 on F(X)), so F(tau) w* lies on the
    triangle: d >= dist(p, F(tau))^2, with equality for the exact variant (Eq.12).  This is what lets
    the GPU drop faces farther than sqrt(kappa delta) from a pixel (Q21)."""
    X0, Y0, _ = _tri(xs[:6])
    X1, Y1, _ = _tri(xs[6:])
    Xt, Yt = (1 - tau) * X0 + tau * X1, (1 - tau) * Y0 + tau * Y1
    det = (Xt[1] - Xt[0]) * (Yt[2] - Yt[0]) - (Yt[1] - Yt[0]) * (Xt[2] - Xt[0])
    if abs(det) < 1e-3:
        return
    w, _ = oracle.bary_textbook(Xt, Yt, u, v)
    if w.min() >= 0:
        return                                          # inside F(tau): not a background term
    true2 = min(_seg_dist2(u, v, Xt[i], Yt[i], Xt[(i + 1) % 3], Yt[(i + 1) % 3]) for i in range(3))
    for exact in (False, True):
        r = oracle.soft_pair(X0, Y0, X1, Y1, tau, u, v, 1e-4, exact=exact)
        assert r is not None
        wh = r["what"]
        assert np.all(wh >= -1e-12) and abs(wh.sum() - 1) < 1e-9
        assert abs(r["d"] - ((r["pstar"][0] - u) ** 2 + (r["pstar"][1] - v) ** 2)) <= 1e-9 * max(1.0, r["d"])
        assert r["d"] >= true2 * (1 - 1e-9) - 1e-12
        if exact:
            assert abs(r["d"] - true2) <= 1e-9 * max(1.0, true2) + 1e-12
