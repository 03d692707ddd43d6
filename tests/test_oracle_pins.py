"""Pins of the fp64 CPU oracle against things other than itself (-m "not gpu").

Each test names what fixes the expected value: a library routine (numpy LU solve, scipy
rotations, sympy adjugate), a closed form, an invariant the paper states, brute force by an
independent numpy renderer, or central finite differences.  A plausible mistake in the
oracle (dropped term, sign, index, transposed operand) fails at least one of them.
"""
import math

import numpy as np
import pytest

import oracle
import scenes

rng0 = np.random.default_rng(7)


# ----------------------------------------------------------------------------- schedule (Q1)

def test_schedule_worked_values():
    # C1: N=8, S=1 -> tau_k = k/7 (P:L235 with K = N)
    s, t = oracle.schedule(8, 1)
    assert np.all(s == 0) and np.allclose(t, np.arange(8) / 7, atol=0, rtol=1e-15)
    # C3: N=50, S=24 (SURVEY Q1 worked values)
    s, t = oracle.schedule(50, 24)
    assert (s[0], t[0]) == (0, 0.0)
    assert s[1] == 0 and t[1] == pytest.approx(24 / 49, abs=1e-15)
    assert s[2] == 0 and t[2] == pytest.approx(48 / 49, abs=1e-15)
    assert s[3] == 1 and t[3] == pytest.approx(23 / 49, abs=1e-15)
    assert (s[49], t[49]) == (23, 1.0)
    # global times reproduce k/(N-1)
    assert np.allclose((s + t) / 24, np.arange(50) / 49, atol=1e-15)
    # PAPER_SEGMENTED 12 x 5: tau in {0, 1/4, 1/2, 3/4, 1} per segment
    s, t = oracle.schedule(60, 12, 1)
    assert np.all(s == np.repeat(np.arange(12), 5))
    assert np.allclose(t, np.tile([0, .25, .5, .75, 1], 12))
    # K = 1 -> 0.5
    s, t = oracle.schedule(12, 12, 1)
    assert np.allclose(t, 0.5) and np.all(s == np.arange(12))
    s, t = oracle.schedule(1, 1)
    assert s[0] == 0 and t[0] == 0.5
    with pytest.raises(ValueError):
        oracle.schedule(10, 3, 1)


# ----------------------------------------------------------------------------- solvers

def _rand_tri(rng, scale=1.0):
    while True:
        x = rng.uniform(-1, 1, 3) * scale
        y = rng.uniform(-1, 1, 3) * scale
        det = np.linalg.det(np.array([x, y, np.ones(3)]))
        if abs(det) > 0.05 * scale * scale:
            return x, y


def test_textbook_solve_matches_lapack():
    rng = np.random.default_rng(1)
    for _ in range(500):
        x, y = _rand_tri(rng)
        u, v = rng.uniform(-1.5, 1.5, 2)
        w, det = oracle.bary_textbook(x, y, u, v)
        F = np.array([x, y, np.ones(3)])
        ref = np.linalg.solve(F, np.array([u, v, 1.0]))     # Eq.3 via LU
        assert np.allclose(w, ref, rtol=0, atol=1e-12 * max(1.0, np.abs(ref).max()))
        assert det == pytest.approx(np.linalg.det(F), rel=1e-12)
        assert abs(w.sum() - 1) < 1e-12                       # homogeneous row of ones
    # vertex and centroid cases
    x, y = np.array([0.1, 0.7, -0.3]), np.array([0.2, -0.4, 0.5])
    w, _ = oracle.bary_textbook(x, y, x[0], y[0])
    assert np.allclose(w, [1, 0, 0], atol=1e-15)
    w, _ = oracle.bary_textbook(x, y, x.mean(), y.mean())
    assert np.allclose(w, [1 / 3] * 3, atol=1e-15)
    # degenerate (Q8)
    w, det = oracle.bary_textbook([0, 1, 2], [0, 1, 2], 0.3, 0.3)
    assert w is None


def test_literal_coefficients_match_sympy_adjugate():
    """A11-A16 as transcribed equal the t-polynomial coefficients of adj(F(t)) p and det F(t),
    derived symbolically here by sympy (independent derivation of Eq.7-8)."""
    sp = pytest.importorskip("sympy")
    t, u, v = sp.symbols("t u v")
    X0 = sp.symbols("x0_0 x1_0 x2_0")
    Y0 = sp.symbols("y0_0 y1_0 y2_0")
    X1 = sp.symbols("x0_1 x1_1 x2_1")
    Y1 = sp.symbols("y0_1 y1_1 y2_1")
    xs = [(1 - t) * X0[i] + t * X1[i] for i in range(3)]
    ys = [(1 - t) * Y0[i] + t * Y1[i] for i in range(3)]
    F = sp.Matrix([xs, ys, [1, 1, 1]])
    num = F.adjugate() * sp.Matrix([u, v, 1])
    den = sp.expand(F.det())
    syms = list(X0) + list(Y0) + list(X1) + list(Y1) + [u, v]
    fnum = [[sp.lambdify(syms, sp.Poly(sp.expand(num[i]), t).coeff_monomial(t ** p)) for p in (2, 1, 0)]
            for i in range(3)]
    fden = [sp.lambdify(syms, sp.Poly(den, t).coeff_monomial(t ** p)) for p in (2, 1, 0)]
    rng = np.random.default_rng(3)
    for _ in range(200):
        a = rng.uniform(-1, 1, 14)
        A1, A2, A3, aa = oracle.fast_coeffs(a[0:3], a[3:6], a[6:9], a[9:12], a[12], a[13])
        for i in range(3):
            assert A1[i] == pytest.approx(fnum[i][0](*a), abs=1e-13)
            assert A2[i] == pytest.approx(fnum[i][1](*a), abs=1e-13)
            assert A3[i] == pytest.approx(fnum[i][2](*a), abs=1e-13)
        for p in range(3):
            assert aa[p] == pytest.approx(fden[p](*a), abs=1e-13)


def test_fast_solver_exact_under_linear_motion():
    """SPEC acceptance 1: Eq.8 == per-t LU solve of the lerped triangle, 1000 instances
    x 101 t, excluding |den| <= 1e-10.  O(1) triangles: 1e-9."""
    rng = np.random.default_rng(4)
    ts = np.linspace(0, 1, 101)
    worst = 0.0
    for _ in range(1000):
        x0, y0 = _rand_tri(rng)
        x1, y1 = _rand_tri(rng)
        u, v = rng.uniform(-1, 1, 2)
        for t in ts:
            w, den = oracle.fast_eval(x0, y0, x1, y1, u, v, t)
            F = np.array([(1 - t) * x0 + t * x1, (1 - t) * y0 + t * y1, np.ones(3)])
            if abs(den) <= 1e-10 or abs(np.linalg.det(F)) < 1e-3:
                continue
            ref = np.linalg.solve(F, [u, v, 1.0])
            worst = max(worst, np.max(np.abs(w - ref)))
    assert worst < 1e-9


def test_coefficient_invariants():
    """sum_i A_pi = a_p; a3 = det F(0); a1+a2+a3 = det F(1);
    static -> A1 = 0, a1 = a2 = 0, A3/a3 = textbook solve; endpoints."""
    rng = np.random.default_rng(5)
    for _ in range(200):
        x0, y0 = _rand_tri(rng)
        x1, y1 = _rand_tri(rng)
        u, v = rng.uniform(-1, 1, 2)
        A1, A2, A3, a = oracle.fast_coeffs(x0, y0, x1, y1, u, v)
        assert A1.sum() == pytest.approx(a[0], abs=1e-13)
        assert A2.sum() == pytest.approx(a[1], abs=1e-13)
        assert A3.sum() == pytest.approx(a[2], abs=1e-13)
        assert a[2] == pytest.approx(np.linalg.det([x0, y0, np.ones(3)]), abs=1e-13)
        assert a.sum() == pytest.approx(np.linalg.det([x1, y1, np.ones(3)]), abs=1e-13)
        assert np.allclose((A1 + A2 + A3) / a.sum(), np.linalg.solve([x1, y1, np.ones(3)], [u, v, 1]), atol=1e-10)
        S1, S2, S3, s = oracle.fast_coeffs(x0, y0, x0, y0, u, v)
        assert np.allclose(S1, 0, atol=1e-15) and abs(s[0]) < 1e-15 and abs(s[1]) < 1e-15
        assert np.allclose(S3 / s[2], np.linalg.solve([x0, y0, np.ones(3)], [u, v, 1]), atol=1e-12)


# ----------------------------------------------------------------------------- projection / pose

def test_projection_closed_forms():
    # camera at (0,0,3) looking at the origin: a vertex on the optical axis projects to the centre,
    # a point at view coords (tan(a), 0, 1) projects to x = 1 (A34)
    ta = math.tan(scenes.HALF_FOV)
    verts = np.array([[0, 0, 0], [ta * 2.0, 0, 1.0], [0, -ta * 0.5, 2.0]], np.float32)
    sc = scenes.single_scene(verts, [[0, 1, 2]], np.ones((3, 3)))
    key, valid, Q = oracle.keyframes(sc)
    assert np.allclose(key[0, 0], [0, 0, 3], atol=1e-7)
    assert key[0, 1, 0] == pytest.approx(1.0, abs=1e-6)       # view z = 2, x = 2 tan(a)
    assert key[0, 2, 1] == pytest.approx(-0.5, abs=1e-6)      # view z = 1, y = -0.5 tan(a)
    assert valid.all()
    # behind the near plane -> invalid
    sc2 = scenes.single_scene([[0, 0, 2.99], [0, 0, 5.0], [1, 0, 0]], [[0, 1, 2]], np.ones((3, 3)))
    _, valid2, _ = oracle.keyframes(sc2)
    assert not valid2[0, 0] and not valid2[0, 1] and valid2[0, 2]


def _look_at(eye, target, up):
    f = np.asarray(target, float) - eye
    f /= np.linalg.norm(f)
    r = np.cross(f, up)
    r /= np.linalg.norm(r)
    return np.stack([r, np.cross(r, f), f])


def _np_keyframes(sc, b):
    """Independent keyframes: scipy rotations + look-at + A34 projection."""
    from scipy.spatial.transform import Rotation
    m = sc.motion
    S = int(m["n_seg"][b])
    cam = sc.cams[b].astype(np.float64)
    R = _look_at(cam[0:3], cam[3:6], cam[6:9])
    ta = math.tan(cam[9])
    P0 = sc.verts.astype(np.float64)
    out = []
    for s in range(S + 1):
        t = s / S
        if m["kind"][b] == 1:
            P = P0 + (t - 0.5) * m["vec"][b].astype(np.float64)
        elif m["kind"][b] in (2, 3):
            ax = m["vec"][b].astype(np.float64)
            rot = Rotation.from_rotvec(ax / np.linalg.norm(ax) * float(m["angle"][b]) * t)
            c = m["pivot"][b].astype(np.float64)
            P = rot.apply(P0 - c) + c
            if m["kind"][b] == 3:                       # A36: T(t) = (s, -4 s^2 + 0.5, s), s = 0.5 - t
                sp = 0.5 - t
                P = P + np.array([sp, -4 * sp * sp + 0.5, sp])
        else:
            P = P0.copy()
        Q = (P - cam[0:3]) @ R.T
        out.append(np.stack([Q[:, 0] / (Q[:, 2] * ta), Q[:, 1] / (Q[:, 2] * ta), Q[:, 2]], -1))
    return np.array(out)


def test_keyframes_match_scipy_rotations():
    sc = scenes.make_c3().subset([0, 3])
    for b in range(2):
        key, valid, _ = oracle.keyframes(sc, b)
        ref = _np_keyframes(sc, b)
        assert np.allclose(key, ref, atol=1e-12)
    # rotation by 2 pi: t = 1 equals t = 0; chord-vs-arc bound
    sc4 = scenes.make_c4().subset([15])
    key, _, _ = oracle.keyframes(sc4, 0)
    # (the angle 2 pi is stored as float32, so the full turn is exact only to ~2e-7 rad)
    assert np.allclose(key[0], key[12], atol=1e-6)


# ----------------------------------------------------------------------------- brute-force renderer

def _np_render(sc, ids_k=-1):
    """Independent brute-force renderer: per pixel, per face (index order), LU solve of the lerped
    screen triangle (Eq.3), inclusive coverage, strict z-test, Eq.9 shading, uniform mean."""
    B, H, W = sc.B, sc.H, sc.W
    out = np.zeros((B, H, W, 4))
    ids = np.full((B, H, W), -1)
    us = -1 + (2 * np.arange(W) + 1) / W
    vs = 1 - (2 * np.arange(H) + 1) / H
    for b in range(B):
        N, S = int(sc.motion["n_sub"][b]), int(sc.motion["n_seg"][b])
        key = _np_keyframes(sc, b)
        zn = sc.cams[b, 10]
        for k in range(N):
            t = 0.5 if N == 1 else k / (N - 1)
            s = min(int(math.floor(t * S + 1e-12)), S - 1) if N > 1 else min(S // 2, S - 1)
            tau = t * S - s
            g = (1 - tau) * key[s] + tau * key[s + 1]
            okv = (key[s][:, 2] > zn) & (key[s + 1][:, 2] > zn)
            for j in range(H):
                for i in range(W):
                    best, bid, bw = np.inf, -1, None
                    for f, fv in enumerate(sc.faces):
                        if not okv[fv].all():
                            continue
                        F = np.array([g[fv, 0], g[fv, 1], np.ones(3)])
                        if abs(np.linalg.det(F)) <= 1e-12:
                            continue
                        w = np.linalg.solve(F, [us[i], vs[j], 1.0])
                        if np.all(w >= 0):
                            z = w @ g[fv, 2]
                            if z < best:
                                best, bid, bw = z, f, w
                    if bid >= 0:
                        out[b, j, i, :3] += bw @ sc.colors[sc.faces[bid]].astype(np.float64)
                        out[b, j, i, 3] += 1
                    if k == ids_k:
                        ids[b, j, i] = bid
        out[b] /= N
    return out, ids


@pytest.mark.parametrize("seed", [11, 12])
def test_oracle_matches_independent_brute_force(seed):
    sc = scenes.random_mesh_scene(12, seed, H=12, W=14)
    ref, rid = _np_render(sc, ids_k=2)
    for mode in ("brute", "binned"):
        r = oracle.render_fwd(sc, mode=mode, ids_k=2, eps_amb=1e-6)
        # ids: bit-exact except where the oracle itself flags the (pixel, k) as Q16-ambiguous
        ok = ~r["amb_ids"]
        assert np.array_equal(r["ids"][ok], rid[ok])
        ok = ~r["amb_img"]
        assert np.max(np.abs(r["rgba"][ok] - ref[ok])) < 1e-12
        assert ok.mean() > 0.9


def test_oracle_rotation_scene_brute_force():
    sc = scenes.random_mesh_scene(10, 21, H=10, W=10,
                                  motion=scenes.rotate((0.3, 1.0, 0.2), 2.0, N=6, S=3))
    ref, rid = _np_render(sc, ids_k=4)
    r = oracle.render_fwd(sc, ids_k=4, eps_amb=1e-6)
    ok = ~r["amb_img"]
    assert np.max(np.abs(r["rgba"][ok] - ref[ok])) < 1e-12
    ok = ~r["amb_ids"]
    assert np.array_equal(r["ids"][ok], rid[ok])


def test_brute_and_binned_bit_identical():
    for sc in (scenes.make_c1(), scenes.make_c2().subset([1])):
        if sc.H > 64:
            sc = scenes.Scene(sc.name, sc.verts, sc.faces, sc.colors, sc.cams, sc.motion, 96, 96)
            sc.motion = {k: v.copy() for k, v in sc.motion.items()}
            sc.motion["n_sub"][:] = 6
        a = oracle.render_fwd(sc, mode="brute", ids_k=1, eps_amb=1e-6)
        b = oracle.render_fwd(sc, mode="binned", ids_k=1, eps_amb=1e-6)
        assert np.array_equal(a["rgba"], b["rgba"])
        assert np.array_equal(a["ids"], b["ids"])
        assert np.array_equal(a["amb_img"], b["amb_img"])
        g = np.random.default_rng(0).normal(size=a["rgba"].shape)
        da = oracle.render_bwd(sc, g, mode="brute")
        db = oracle.render_bwd(sc, g, mode="binned")
        assert np.array_equal(da[0], db[0]) and np.array_equal(da[1], db[1])


# ----------------------------------------------------------------------------- closed forms

def test_full_frame_triangle_constant_colour():
    """one triangle filling the frame with uniform colour c -> every pixel rgb = c, alpha 1."""
    c = np.array([0.2, 0.5, 0.7])
    verts = [[-10, -10, 0], [10, -10, 0], [0, 10, 0]]
    sc = scenes.single_scene(verts, [[0, 1, 2]], [c, c, c], H=9, W=11)
    r = oracle.render_fwd(sc)
    assert np.allclose(r["rgba"][..., :3], c, atol=1e-14)
    assert np.all(r["rgba"][..., 3] == 1.0)


def test_parallel_planes_nearer_wins():
    """two parallel triangles at depth 1 and 2 -> the nearer wins where both cover."""
    big = np.array([[-3, -3], [3, -3], [0, 3]])
    verts = np.concatenate([np.c_[big, np.full(3, 1.0)], np.c_[big * 0.5, np.full(3, 2.0)]])  # z world
    # camera at z = 3 looking at -z: world z=2 is nearer (view depth 1) than z=1 (view depth 2)
    sc = scenes.single_scene(verts, [[0, 1, 2], [3, 4, 5]], np.r_[np.zeros((3, 3)), np.ones((3, 3))],
                             H=8, W=8)
    r = oracle.render_fwd(sc, ids_k=0)
    # both project to the same screen triangle (similar triangles); the near one wins wherever covered
    cov = r["ids"][0] >= 0
    assert cov.mean() > 0.8 and np.all(r["ids"][0][cov] == 1)
    assert np.allclose(r["rgba"][0][cov][:, :3], 1.0)
    sc2 = scenes.single_scene(verts, [[3, 4, 5], [0, 1, 2]], np.r_[np.ones((3, 3)), np.zeros((3, 3))],
                              H=8, W=8)
    r2 = oracle.render_fwd(sc2, ids_k=0)
    assert np.all(r2["ids"][0][r2["ids"][0] >= 0] == 0)


def test_interpenetrating_pair_matches_plane_depths():
    """interpenetrating triangles; winner = nearer of the two planes, computed per pixel
    from the analytic view depths of the two planes (no barycentrics involved)."""
    ta = math.tan(scenes.HALF_FOV)
    # two planes in view space: z = 2 + 0.5 x  and z = 2 - 0.5 x (cross at x = 0), big triangles
    def tri(sl):
        pts = []
        for (xn, yn) in [(-1.5, -1.5), (1.5, -1.5), (0.0, 1.5)]:
            # ray through NDC (xn, yn): view point = z (xn ta, yn ta, 1); plane z = 2 + sl * x_view
            z = 2.0 / (1.0 - sl * xn * ta)
            pts.append([z * xn * ta, z * yn * ta, 3.0 - z])   # world (camera at z=3 looking -z)
        return pts
    verts = np.array(tri(0.5) + tri(-0.5))
    sc = scenes.single_scene(verts, [[0, 1, 2], [3, 4, 5]], np.r_[np.zeros((3, 3)), np.ones((3, 3))],
                             H=10, W=11)
    r = oracle.render_fwd(sc, ids_k=0, eps_amb=1e-6)
    us = -1 + (2 * np.arange(11) + 1) / 11
    for j in range(10):
        for i in range(11):
            xn = us[i]
            z0 = 2.0 / (1.0 - 0.5 * xn * ta)
            z1 = 2.0 / (1.0 + 0.5 * xn * ta)
            exp = 0 if z0 < z1 else 1
            if r["ids"][0, j, i] >= 0 and not r["amb_ids"][0, j, i]:
                assert r["ids"][0, j, i] == exp


def _square_scene(N, T, H=8, W=32, half=0.3):
    verts = [[-half, -half, 0], [half, -half, 0], [half, half, 0], [-half, half, 0]]
    return scenes.single_scene(verts, [[0, 1, 2], [0, 2, 3]], np.full((4, 3), 0.6),
                               motion=scenes.translate(T, N=N), H=H, W=W)


def test_translating_square_alpha_counts():
    """A screen-aligned square translating along x, camera on the z axis: depth is constant, so the
    screen lerp is exact and alpha(pixel) = #{k : |u - x_c(t_k)| <= half_ndc} / N, counted by hand;
    rgb = 0.6 alpha."""
    N, T, half = 9, (1.2, 0, 0), 0.3
    sc = _square_scene(N, T, half=half)
    r = oracle.render_fwd(sc, eps_amb=1e-6)
    ta = math.tan(scenes.HALF_FOV)
    sc_ndc = 1.0 / (3.0 * ta)             # world -> NDC at depth 3
    us = -1 + (2 * np.arange(32) + 1) / 32
    vs = 1 - (2 * np.arange(8) + 1) / 8
    for j in range(8):
        for i in range(32):
            if abs(vs[j]) > half * sc_ndc:
                cnt = 0
            else:
                cnt = sum(abs(us[i] - (k / (N - 1) - 0.5) * T[0] * sc_ndc) <= half * sc_ndc for k in range(N))
            if not r["amb_img"][0, j, i]:
                assert r["rgba"][0, j, i, 3] == pytest.approx(cnt / N, abs=1e-14)
                c32 = float(np.float32(0.6))          # colours are stored as float32
                assert r["rgba"][0, j, i, 0] == pytest.approx(c32 * cnt / N, abs=1e-12)


def test_n1_is_static_render_at_half():
    """N=1 -> the single sample at tau = 0.5.  With a translation parallel to the image plane
    (camera on the z axis) the screen lerp is exact, so this is a static render of the mid pose."""
    sc = scenes.random_mesh_scene(15, 31, H=16, W=16, motion=scenes.translate((0.7, -0.2, 0.0), N=1))
    mid = scenes.random_mesh_scene(15, 31, H=16, W=16, motion=scenes.static(1))
    a = oracle.render_fwd(sc)["rgba"]
    b = oracle.render_fwd(mid)["rgba"]       # translate at t=0.5 is the identity placement
    assert np.max(np.abs(a - b)) < 1e-12


def test_zero_motion_equals_static():
    """a static trajectory renders identically for any N."""
    a = oracle.render_fwd(scenes.random_mesh_scene(15, 41, motion=scenes.translate((0, 0, 0), N=7)))
    b = oracle.render_fwd(scenes.random_mesh_scene(15, 41, motion=scenes.static(1)))
    assert np.max(np.abs(a["rgba"] - b["rgba"])) < 1e-14


def test_blur_is_mean_of_exact_pose_renders_for_x_translation():
    """Closed-form special case: x-translation seen from a camera on the z axis keeps
    every vertex depth constant, so the screen lerp is exact and the blurred image equals the mean
    of N static renders at the exact poses t_k (S:L296 linearity)."""
    N, T = 6, np.array([0.9, 0.0, 0.0], np.float32).astype(np.float64)   # motion params are float32
    sc = scenes.random_mesh_scene(10, 51, H=14, W=14, motion=scenes.translate(T, N=N))
    blur = oracle.render_fwd(sc)["rgba"]
    acc = np.zeros_like(blur)
    for k in range(N):
        shifted = scenes.random_mesh_scene(10, 51, H=14, W=14, motion=scenes.static(1))
        shifted.verts = (shifted.verts.astype(np.float64) + (k / (N - 1) - 0.5) * T)
        acc += oracle.render_fwd(shifted)["rgba"]
    assert np.max(np.abs(blur - acc / N)) < 1e-9


def test_fast_solver_cross_check_in_oracle():
    r = oracle.render_fwd(scenes.make_c1(), check_fast=True)
    st = r["stats"]
    assert st["n_checked"] == st["necessary_pairs"] > 1000
    assert st["max_fast_dev"] < 1e-6


def test_behind_camera_flag():
    sc = scenes.single_scene([[0, 0, 2.99], [1, 0, 0], [0, 1, 0], [-1, 0, 0], [0, -1, 0], [0.2, 0.2, 0]],
                             [[0, 1, 2], [3, 4, 5]], np.ones((6, 3)))
    r = oracle.render_fwd(sc, ids_k=0)
    assert r["behind"]
    assert not np.any(r["ids"] == 0)          # faces with a behind-camera vertex are skipped


# ----------------------------------------------------------------------------- backward

def _frozen_loss(sc, G, frozen, verts=None, colors=None):
    return float(np.sum(G * oracle.render_fwd(sc, frozen=frozen, verts=verts, colors=colors)["rgba"]))


def _winners(sc):
    N = int(sc.motion["n_sub"][0])
    fz = np.zeros((N, sc.H, sc.W), np.int32)
    for k in range(N):
        fz[k] = oracle.render_fwd(sc, ids_k=k)["ids"][0]
    return fz.reshape(-1)


@pytest.mark.parametrize("motion", [scenes.translate((0.6, 0.2, -0.4), N=5),
                                    scenes.rotate((0.2, 1, 0.1), 1.5, N=7, S=3)])
def test_backward_matches_frozen_visibility_fd(motion):
    """Frozen-visibility central differences (SURVEY 8(c) backward pin): the derivative
    the method defines.  h = 1e-6 in fp64."""
    sc = scenes.random_mesh_scene(8, 61, H=12, W=12, motion=motion)
    G = np.random.default_rng(2).normal(size=(1, 12, 12, 4))
    fz = _winners(sc)
    dv, dc = oracle.render_bwd(sc, G)
    V = sc.V
    V64 = sc.verts.astype(np.float64)
    h = 1e-6
    num = np.zeros((V, 3))
    for v in range(V):
        for c in range(3):
            vp, vm = V64.copy(), V64.copy()
            vp[v, c] += h
            vm[v, c] -= h
            num[v, c] = (_frozen_loss(sc, G, fz, verts=vp) - _frozen_loss(sc, G, fz, verts=vm)) / (2 * h)
    assert np.linalg.norm(dv - num) / np.linalg.norm(num) < 1e-6
    # colour gradient: the loss is linear in colours -> FD exact up to rounding
    C64 = sc.colors.astype(np.float64)
    numc = np.zeros((V, 3))
    for v in range(V):
        for c in range(3):
            cp, cm = C64.copy(), C64.copy()
            cp[v, c] += 1e-3
            cm[v, c] -= 1e-3
            numc[v, c] = (_frozen_loss(sc, G, fz, colors=cp) - _frozen_loss(sc, G, fz, colors=cm)) / 2e-3
    assert np.max(np.abs(dc - numc)) < 1e-9


def test_backward_linearity_and_separability():
    """zero seed -> zero; linear in the seed; red-only seed -> only red colour
    gradients; alpha-only seed -> no gradient (hard coverage)."""
    sc = scenes.random_mesh_scene(12, 71, H=12, W=12, motion=scenes.translate((0.5, 0.1, 0.0), N=4))
    g = np.random.default_rng(3).normal(size=(1, 12, 12, 4))
    z = oracle.render_bwd(sc, np.zeros_like(g))
    assert not np.any(z[0]) and not np.any(z[1])
    a = oracle.render_bwd(sc, g)
    b = oracle.render_bwd(sc, 2.5 * g)
    assert np.allclose(b[0], 2.5 * a[0], rtol=1e-12, atol=1e-14)
    assert np.allclose(b[1], 2.5 * a[1], rtol=1e-12, atol=1e-14)
    gr = np.zeros_like(g)
    gr[..., 0] = g[..., 0]
    r = oracle.render_bwd(sc, gr)
    assert np.any(r[1][:, 0]) and not np.any(r[1][:, 1:])
    ga = np.zeros_like(g)
    ga[..., 3] = 1.0
    r = oracle.render_bwd(sc, ga)
    assert not np.any(r[0]) and not np.any(r[1])


def test_pixel_list_mode_matches_full():
    sc = scenes.make_c1()
    full = oracle.render_fwd(sc, ids_k=3)
    pix = np.array([[0, 20, 30], [0, 32, 32], [0, 5, 60], [0, 40, 12]])
    r = oracle.render_fwd(sc, pixels=pix, ids_k=3)
    for q, (b, j, i) in enumerate(pix):
        assert np.array_equal(r["rgba"][q], full["rgba"][b, j, i])
        assert r["ids"][q] == full["ids"][b, j, i]
    G = np.zeros((1, 64, 64, 4))
    Gp = np.random.default_rng(0).normal(size=(4, 4))
    for q, (b, j, i) in enumerate(pix):
        G[b, j, i] = Gp[q]
    a = oracle.render_bwd(sc, G)
    b = oracle.render_bwd(sc, Gp, pixels=pix)
    assert np.allclose(a[0], b[0], atol=1e-13) and np.allclose(a[1], b[1], atol=1e-13)


# ----------------------------------------------------------------------------- NEXT-3 motions

def test_parabolic_pose_midpoint():
    """S:L82 / A35-A37: at t = 0.5 the parabolic composite is a rotation by pi/2 about y plus the
    translation (0, 0.5, 0); keyframes match the independent scipy construction at every t = s/S."""
    sc = scenes.random_mesh_scene(6, 81, motion=scenes.parabolic(N=5, S=4))
    sc.cams[0, 0:3] = [0.3, 0.2, 4.0]
    key, valid, Q = oracle.keyframes(sc, 0)
    assert np.allclose(key, _np_keyframes(sc, 0), atol=1e-12)
    P0 = sc.verts.astype(np.float64)
    mid = np.stack([P0[:, 2], P0[:, 1] + 0.5, -P0[:, 0]], 1)     # R_y(pi/2) (x, y, z) = (z, y, -x)
    R = _look_at(sc.cams[0, 0:3].astype(np.float64), [0, 0, 0], [0, 1, 0])
    Qm = (mid - sc.cams[0, 0:3].astype(np.float64)) @ R.T
    assert np.allclose(Q[2], Qm, atol=1e-6)       # float32 angle pi


def test_exact_pose_reference_is_mean_of_static_renders():
    """NEXT-3 reference: N sub-frames on N-1 segments sample the exact rigid poses, so the blurred
    image equals the mean of N static renders of the mesh posed (by scipy) at t_k = k/(N-1)."""
    from scipy.spatial.transform import Rotation
    N = 5
    sc = scenes.random_mesh_scene(10, 91, H=14, W=14,
                                  motion=scenes.exact_pose(scenes.rotate((0.1, 1.0, 0.2), 2.5, N=N, S=1)))
    blur = oracle.render_fwd(sc)["rgba"]
    acc = np.zeros_like(blur)
    ax = sc.motion["vec"][0].astype(np.float64)
    for k in range(N):
        rot = Rotation.from_rotvec(ax / np.linalg.norm(ax) * float(sc.motion["angle"][0]) * k / (N - 1))
        st = scenes.random_mesh_scene(10, 91, H=14, W=14, motion=scenes.static(1))
        st.verts = rot.apply(st.verts.astype(np.float64))
        acc += oracle.render_fwd(st)["rgba"]
    assert np.max(np.abs(blur - acc / N)) < 1e-9


def test_segmentation_converges_to_exact_pose():
    """Appendix 'Segmentation Analysis': more linear segments approach the
    exact-pose render (monotone PSNR on a spinning mesh)."""
    base = scenes.random_mesh_scene(30, 93, H=24, W=24, motion=scenes.rotate((0, 1, 0), 2 * math.pi, N=48, S=1))
    ref = oracle.render_fwd(dataclasses_replace_motion(base, scenes.exact_pose(scenes.rotate((0, 1, 0), 2 * math.pi,
                                                                                             N=48, S=1))))["rgba"]
    psnr = []
    for S in (3, 6, 12, 24):
        img = oracle.render_fwd(dataclasses_replace_motion(base, scenes.rotate((0, 1, 0), 2 * math.pi, N=48,
                                                                               S=S)))["rgba"]
        mse = np.mean((img[..., :3] - ref[..., :3]) ** 2)
        psnr.append(10 * np.log10(1.0 / max(mse, 1e-30)))
    assert all(b > a for a, b in zip(psnr, psnr[1:])), psnr


def dataclasses_replace_motion(sc, motion):
    import dataclasses
    return dataclasses.replace(sc, motion=scenes.motion_arrays([motion] * sc.B))


def test_automatic_segment_count_rule():
    """Q24 (n_seg = 0): one segment for translation, 12 per full turn for rotation."""
    import dataclasses
    sc = scenes.random_mesh_scene(3, 4, motion=scenes.rotate((0, 1, 0), 2 * math.pi * 1.5, N=10, S=0))
    assert oracle.segments(sc) == 18
    sc2 = scenes.random_mesh_scene(3, 4, motion=scenes.translate((1, 0, 0), N=10, S=0))
    assert oracle.segments(sc2) == 1
    sc3 = scenes.random_mesh_scene(3, 4, motion=scenes.rotate((0, 1, 0), 0.3, N=10, S=0))
    assert oracle.segments(sc3) == 1
    # rendering with S = 0 equals rendering with the resolved count
    m = dict(sc.motion)
    m["n_seg"] = np.array([18], np.int32)
    a = oracle.render_fwd(sc)["rgba"]
    b = oracle.render_fwd(dataclasses.replace(sc, motion=m))["rgba"]
    assert np.array_equal(a, b)
