"""Pins of the oracle's parity exclusion masks (Q16/Q18) and of the translation's time direction.

The masks gate every GPU parity comparison, so they are pinned here against geometry whose answer is
known by construction, not against the oracle itself:
  * amb_ids  the winner at sub-frame ids_k can change when every inside test moves by eps = 1e-6 NDC of
             signed edge distance (loose: -eps, strict: +eps, watertight across shared edges) or under a
             depth tie within 1e-6 relative (north_star: "bit-exact except at pixels within 1e-6 of an
             edge or depth tie"; P:L221 coverage rule);
  * amb_img  those perturbations can move the blurred value by more than 1e-5;
  * amb_win  the winner can change at some sub-frame (the gradient comparison's exclusion, Q18).
Scenes: a camera at (0, 0, 1) looking down -z with half field of view 45 degrees and vertices at z = 0,
so a vertex's NDC x is its world x (A34: x / (z tan alpha) with z = tan alpha = 1), and
pixel centres at (-1 + (2i+1)/W, 1 - (2j+1)/H) (Q9).  Vertical edges are placed at signed distances
{-2, -0.5, 0, +0.5, +2} eps from the centres of one pixel column.  A mutation that widens eps to 1e-3
flags the 2-eps pixels and fails these pins (test_wider_eps_is_detected shows it does).
"""
import math

import numpy as np
import pytest

import oracle
import scenes

EPS = 1e-6                      # DESIGN.md Q16: signed NDC edge distance
ZTIE = 1e-6                     # DESIGN.md Q16: relative depth tie
H = W = 8
COL = 4                         # test column, u = 0.125
U = -1 + (2 * np.arange(W) + 1) / W
V = 1 - (2 * np.arange(H) + 1) / H
CAM = scenes.camera_row((0, 0, 1), half_fov=math.pi / 4, z_near=0.05)


def _scene(verts, faces, colors, motion=None):
    return scenes.single_scene(verts, faces, colors, cam=CAM, motion=motion, H=H, W=W)


def _seg_dist(px, py, a, b):
    """Euclidean distance from (px, py) to the segment a-b (independent fp64 geometry)."""
    a, b = np.asarray(a, float), np.asarray(b, float)
    d = b - a
    t = np.clip(((px - a[0]) * d[0] + (py - a[1]) * d[1]) / (d @ d), 0.0, 1.0)
    return math.hypot(px - a[0] - t * d[0], py - a[1] - t * d[1])


def _near_segments(segs, eps=EPS):
    """Pixels within eps of some segment ((x, y), (x, y))."""
    m = np.zeros((H, W), bool)
    for a, b in segs:
        for j in range(H):
            for i in range(W):
                if _seg_dist(U[i], V[j], a[:2], b[:2]) < eps:
                    m[j, i] = True
    return m


def _near_edge(tris, eps=EPS):
    """Pixels within eps of some edge of some triangle (2-D NDC vertex triples)."""
    return _near_segments([(tri[k], tri[(k + 1) % 3]) for tri in tris for k in range(3)], eps)


def _flags(sc, eps=EPS, ids_k=0):
    r = oracle.render_fwd(sc, mode="brute", ids_k=ids_k, eps_amb=eps)
    return r, r["amb_ids"][0], r["amb_img"][0], r["amb_win"][0]


def _edge_x(s):
    """fp32 vertex x of a vertical edge at signed distance s from the test column's centres (s > 0: the
    centres are to the right of the edge) and the exact distance the fp32 rounding leaves."""
    e = np.float32(U[COL] - s)
    return e, U[COL] - float(e)


@pytest.mark.parametrize("s", [2 * EPS, 0.5 * EPS, 0.0, -0.5 * EPS, -2 * EPS])
def test_lone_edge_flags(s):
    """One triangle to the right of a vertical boundary edge (no neighbour).  Centres within eps of the
    edge flag all three masks (strict drops the face inside, loose adds it outside: coverage, hence
    alpha, changes by 1 at N = 1); centres 2 eps away, and every other pixel, flag none."""
    e, d = _edge_x(s)
    tri = [(e, -0.9, 0), (e, 0.9, 0), (0.9, 0.0, 0)]
    sc = _scene(tri, [[0, 1, 2]], np.full((3, 3), 0.7))
    r, ids, img, win = _flags(sc)
    exp = _near_edge([tri])
    assert exp[3, COL] == exp[4, COL] == (abs(d) < EPS)
    assert np.array_equal(ids, exp) and np.array_equal(img, exp) and np.array_equal(win, exp)
    # the nominal coverage itself follows the sign of d (inclusive at 0)
    if abs(d) >= 0.4 * EPS:
        assert (r["rgba"][0, 3, COL, 3] == 1.0) == (d > 0)


@pytest.mark.parametrize("s", [2 * EPS, 0.5 * EPS, 0.0, -0.5 * EPS, -2 * EPS])
@pytest.mark.parametrize("crease", [0.0, 0.4])
def test_shared_edge_flags(s, crease):
    """Two faces sharing a vertical interior edge (same two vertex indices), coplanar or creased (the
    left face's far vertex pushed back): depth is continuous across the edge, so within eps of it the
    loose scenario adds the neighbour at a tied depth and the winning face can change (amb_ids,
    amb_win); at 2 eps neither perturbation reaches the neighbour: no flag.  The value cannot change:
    the strict scenario is watertight (it keeps a face whose neighbour covers the pixel from the other
    side, so no background crack opens) and the two faces' shading agrees on the edge (shared vertices,
    shared colours; Eq.9), so amb_img stays clear there.  The boundary edges flag as in the lone case."""
    e, d = _edge_x(s)
    verts = [(e, -0.9, 0), (e, 0.9, 0), (0.9, 0.0, 0), (-0.9, 0.0, -crease)]
    cols = np.array([[0.2, 0.8, 0.1], [0.2, 0.8, 0.1], [0.2, 0.8, 0.1], [0.9, 0.1, 0.3]])
    sc = _scene(verts, [[0, 1, 2], [1, 0, 3]], cols)
    r, ids, img, win = _flags(sc)
    # the creased face projects its far vertex at x / (1 + crease) (A34)
    xl = -0.9 / (1 + crease)
    exp = _near_edge([[(e, -0.9), (e, 0.9), (0.9, 0.0)], [(e, -0.9), (e, 0.9), (xl, 0.0)]])
    boundary = _near_segments([((e, 0.9), (0.9, 0.0)), ((0.9, 0.0), (e, -0.9)), ((e, 0.9), (xl, 0.0)),
                               ((xl, 0.0), (e, -0.9))])
    assert exp[3, COL] == (abs(d) < EPS)
    assert np.array_equal(ids, exp) and np.array_equal(win, exp)
    assert np.array_equal(img, boundary)
    assert r["rgba"][0, 3, COL, 3] == 1.0 and r["rgba"][0, 4, COL, 3] == 1.0   # no crack, any d


def _overlap_scene(dz, same_colour=False):
    """Face 0 at z = 0 and an overlapping face 1 (other vertices) at z = dz: view depths 1 and 1 - dz."""
    verts = [(-0.95, -0.95, 0), (0.95, -0.95, 0), (0.0, 0.95, 0),
             (-0.9, -0.85, dz), (0.85, -0.9, dz), (0.05, 0.9, dz)]
    cols = np.array([[0.9, 0.1, 0.1]] * 3 + [[0.9, 0.1, 0.1] if same_colour else [0.1, 0.9, 0.1]] * 3)
    tris = [[(-0.95, -0.95), (0.95, -0.95), (0.0, 0.95)],
            [(x / (1 - dz), y / (1 - dz)) for x, y, _ in verts[3:]]]
    return _scene(verts, [[0, 1, 2], [3, 4, 5]], cols), tris


@pytest.mark.parametrize("dz,tie", [(0.0, True), (0.5e-6, True), (2e-6, False), (1e-3, False)])
def test_depth_tie_flags(dz, tie):
    """Overlapping faces (no shared edge) at relative depth difference dz: inside both and away from
    edges the winner can change iff |dz| <= 1e-6 (Q16 depth tie); a tie-free scene flags nothing but
    the pixels within eps of an edge."""
    sc, tris = _overlap_scene(dz)
    r, ids, img, win = _flags(sc)
    near = _near_edge(tris)
    both = np.zeros((H, W), bool)
    for j in range(H):
        for i in range(W):
            both[j, i] = all(_inside(U[i], V[j], t) for t in tris)
    exp = near | (both & tie)
    assert both.sum() >= 20
    assert np.array_equal(ids, exp) and np.array_equal(win, exp) and np.array_equal(img, exp)
    if not tie:   # the nearer face (smaller view depth) wins
        assert np.all(r["ids"][0][both & ~near] == (1 if dz > 0 else 0))


def test_tie_between_equal_shades_moves_ids_not_values():
    """amb_ids and amb_img differ: a depth tie between faces of equal colour can change the winning
    face (amb_ids) but not the blurred value (amb_img needs a change > 1e-5)."""
    sc, tris = _overlap_scene(0.0, same_colour=True)
    _, ids, img, win = _flags(sc)
    near = _near_edge(tris)
    both = np.array([[all(_inside(U[i], V[j], t) for t in tris) for i in range(W)] for j in range(H)])
    assert np.array_equal(ids, near | both) and np.array_equal(win, near | both)
    assert np.array_equal(img, near)


def _inside(px, py, tri):
    (x0, y0), (x1, y1), (x2, y2) = tri
    d = (x1 - x0) * (y2 - y0) - (x2 - x0) * (y1 - y0)
    w1 = ((px - x0) * (y2 - y0) - (x2 - x0) * (py - y0)) / d
    w2 = ((x1 - x0) * (py - y0) - (px - x0) * (y1 - y0)) / d
    return min(w1, w2, 1 - w1 - w2) >= 0.0


def test_amb_win_covers_other_subframes():
    """amb_win flags a pixel whose winner is ambiguous at any sub-frame, amb_ids only at ids_k: a
    triangle translating along x whose edge passes 0.5 eps from the test column at the middle
    sub-frame (t = 0.5, P(t) = P0 + (t - 0.5) T: the rest pose) and far from it at t = 0 and t = 1."""
    e, d = _edge_x(0.5 * EPS)
    tri = [(e, -0.9, 0), (e, 0.9, 0), (0.9, 0.0, 0)]
    sc = _scene(tri, [[0, 1, 2]], np.full((3, 3), 0.7), motion=scenes.translate((0.2, 0, 0), N=3))
    _, ids0, img0, win0 = _flags(sc, ids_k=0)
    _, ids1, _, win1 = _flags(sc, ids_k=1)
    assert win0[3, COL] and win1[3, COL] and ids1[3, COL]
    assert not ids0[3, COL]
    assert img0[3, COL]       # one sub-frame's alpha can change by 1: 1/3 of the blurred value


def test_wider_eps_is_detected():
    """The mutation eps = 1e-3 flags the 2-eps pixels: the pins above would fail under it."""
    e, _ = _edge_x(2 * EPS)
    tri = [(e, -0.9, 0), (e, 0.9, 0), (0.9, 0.0, 0)]
    sc = _scene(tri, [[0, 1, 2]], np.full((3, 3), 0.7))
    _, ids, _, _ = _flags(sc, eps=1e-3)
    assert ids[3, COL] and not np.array_equal(ids, _near_edge([tri]))


@pytest.mark.parametrize("k,x_c", [(0, 0.5), (2, -0.5)])
def test_translation_time_direction(k, x_c):
    """A30: x(t) = x0 + (0.5 - t), "from x0 + 0.5 at t = 0 to x0 - 0.5 at t = 1".  A
    rectangle of half-width 0.1 (half-height 0.3) at x0 = 0 with T = (-1, 0, 0) (the paper's translation),
    N = 3 sub-frames t = 0, 0.5, 1, rendering only sub-frame k (sub_range [k, k+1)): alpha = 1/3 on the
    pixels whose centre lies within the rectangle at x_c = x0 + (0.5 - t_k), 0 elsewhere."""
    half, hh, Wd = 0.1, 0.3, 40
    verts = [(-half, -hh, 0), (half, -hh, 0), (half, hh, 0), (-half, hh, 0)]
    sc = scenes.single_scene(verts, [[0, 1, 2], [0, 2, 3]], np.full((4, 3), 0.5), cam=CAM,
                             motion=scenes.translate((-1.0, 0, 0), N=3), H=8, W=Wd)
    r = oracle.render_fwd(sc, sub_range=[[k, k + 1]])
    us = -1 + (2 * np.arange(Wd) + 1) / Wd
    vs = 1 - (2 * np.arange(8) + 1) / 8
    for j in range(8):
        for i in range(Wd):
            inside = abs(us[i] - x_c) < half - 1e-9 and abs(vs[j]) < hh - 1e-9
            outside = abs(us[i] - x_c) > half + 1e-9 or abs(vs[j]) > hh + 1e-9
            a = r["rgba"][0, j, i, 3]
            if inside:
                assert a == pytest.approx(1 / 3, abs=1e-12)
            elif outside:
                assert a == 0.0
    assert r["rgba"][0, 3:5, :, 3].sum() > 0
