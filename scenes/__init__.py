"""Seeded synthetic input generators for the motion-blur hot path.

This module is shared by the CUDA path (tests, bench, smoke) and by the CPU
oracle's tests.  It holds NONE of the method's arithmetic: no projection, no
barycentric solve, no schedule, no shading.  It only builds meshes, colours,
camera placements, motion parameters and loss targets, with the shapes,
sizes and value distributions of SURVEY.md section 8(d) (configs C1-C5 of
BASELINE.json).  The paper's own workloads (ShapeNet models, P:L457-458,
P:L1467) are not in the container; these meshes stand in for them.

Array conventions (consumed identically by both sides):
  verts   float32 [V,3]   world positions P0
  faces   int32   [F,3]   vertex indices
  colors  float32 [V,3]   per-vertex RGB in [0,1]
  cams    float32 [B,11]  eye(3) target(3) up(3) half_fov(rad) z_near
  motion  dict of arrays, one entry per image b:
          kind int32[B] (0 static, 1 translate, 2 rotate), vec f32[B,3]
          (translation T over the exposure, or unit rotation axis),
          angle f32[B] (total rotation angle), pivot f32[B,3],
          n_sub int32[B] (N), n_seg int32[B] (S), rule int32[B]
          (0 GLOBAL_INCLUSIVE, 1 PAPER_SEGMENTED)
  target  float32 [B,H,W,4] loss target (RGBA)
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

import numpy as np

STATIC, TRANSLATE, ROTATE, PARABOLIC = 0, 1, 2, 3
GLOBAL_INCLUSIVE, PAPER_SEGMENTED = 0, 1

HALF_FOV = math.radians(30.0)      # A34, P:L1455 ("fixed half-angular field of view alpha = 30 deg")
CAM_DIST = 2.232                   # A33
Z_NEAR = 0.05
MASTER_SEED = 20261019             # seed = 20261019 + config index


@dataclasses.dataclass
class Scene:
    name: str
    verts: np.ndarray
    faces: np.ndarray
    colors: np.ndarray
    cams: np.ndarray
    motion: dict
    H: int
    W: int
    target: Optional[np.ndarray] = None
    meta: dict = dataclasses.field(default_factory=dict)

    @property
    def B(self) -> int:
        return int(self.cams.shape[0])

    @property
    def V(self) -> int:
        return int(self.verts.shape[0])

    @property
    def F(self) -> int:
        return int(self.faces.shape[0])

    def subset(self, images) -> "Scene":
        """Scene restricted to a list of image indices (mesh shared)."""
        idx = np.asarray(images, dtype=np.int64)
        mo = {k: np.ascontiguousarray(v[idx]) for k, v in self.motion.items()}
        tgt = None if self.target is None else np.ascontiguousarray(self.target[idx])
        return dataclasses.replace(self, cams=np.ascontiguousarray(self.cams[idx]),
                                   motion=mo, target=tgt)

    def save(self, path: str) -> None:
        arrs = dict(verts=self.verts, faces=self.faces, colors=self.colors,
                    cams=self.cams, H=np.int64(self.H), W=np.int64(self.W))
        for k, v in self.motion.items():
            arrs["motion_" + k] = v
        if self.target is not None:
            arrs["target"] = self.target
        np.savez_compressed(path, **arrs)


# --------------------------------------------------------------------------- meshes

def icosphere(level: int, radius: float = 1.0):
    """Icosahedron subdivided `level` times (midpoint split, re-normalised).
    Level 1: 42 V / 80 F; 3: 642 / 1,280; 5: 10,242 / 20,480; 6: 40,962 / 81,920
    (SURVEY Q15)."""
    t = (1.0 + 5.0 ** 0.5) / 2.0
    v = [(-1, t, 0), (1, t, 0), (-1, -t, 0), (1, -t, 0), (0, -1, t), (0, 1, t),
         (0, -1, -t), (0, 1, -t), (t, 0, -1), (t, 0, 1), (-t, 0, -1), (-t, 0, 1)]
    f = [(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11), (1, 5, 9), (5, 11, 4),
         (11, 10, 2), (10, 7, 6), (7, 1, 8), (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8),
         (3, 8, 9), (4, 9, 5), (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1)]
    verts = [np.array(p, dtype=np.float64) / np.linalg.norm(p) for p in v]
    faces = f
    for _ in range(level):
        cache = {}
        nf = []

        def mid(a, b):
            key = (a, b) if a < b else (b, a)
            if key not in cache:
                m = verts[a] + verts[b]
                verts.append(m / np.linalg.norm(m))
                cache[key] = len(verts) - 1
            return cache[key]

        for (a, b, c) in faces:
            ab, bc, ca = mid(a, b), mid(b, c), mid(c, a)
            nf += [(a, ab, ca), (b, bc, ab), (c, ca, bc), (ab, bc, ca)]
        faces = nf
    V = np.array(verts) * radius
    return V, np.array(faces, dtype=np.int32)


def revolution_top(rng: np.random.Generator, n_profile: int = 64, n_azimuth: int = 80):
    """Spinning-top surface of revolution: n_profile rings of
    n_azimuth vertices (pole rings collapse to a point, kept as duplicate vertices),
    two triangles per quad, degenerate pole triangles dropped.
    64 x 80 -> 5,120 V / 9,920 F.  Returns verts (about the y axis), faces, azimuth index."""
    s = np.linspace(0.0, 1.0, n_profile)
    coef = rng.normal(size=(3, 2)) / np.arange(1, 4)[:, None]
    four = sum(coef[m, 0] * np.cos(2 * np.pi * (m + 1) * s) + coef[m, 1] * np.sin(2 * np.pi * (m + 1) * s)
               for m in range(3))
    env = np.sin(np.pi * s) ** 0.7 * (1.25 - 0.7 * s)        # wide body, pointed tip at s=0
    r = 0.8 * env * (1.0 + 0.05 * four)
    r[0] = r[-1] = 0.0
    y = 2.0 * s - 1.0
    phi = 2 * np.pi * np.arange(n_azimuth) / n_azimuth
    X = r[:, None] * np.cos(phi)[None, :]
    Z = r[:, None] * np.sin(phi)[None, :]
    Y = np.broadcast_to(y[:, None], X.shape)
    verts = np.stack([X, Y, Z], -1).reshape(-1, 3)
    az = np.broadcast_to(np.arange(n_azimuth)[None, :], X.shape).reshape(-1)
    faces = []
    for i in range(n_profile - 1):
        for j in range(n_azimuth):
            a = i * n_azimuth + j
            b = i * n_azimuth + (j + 1) % n_azimuth
            c = (i + 1) * n_azimuth + j
            d = (i + 1) * n_azimuth + (j + 1) % n_azimuth
            if i != 0:                   # (a, b) on the bottom pole ring would be degenerate
                faces.append((a, b, d))
            if i != n_profile - 2:       # (c, d) on the top pole ring would be degenerate
                faces.append((a, d, c))
    verts = verts / np.max(np.linalg.norm(verts, axis=1))   # max norm 1
    return verts, np.array(faces, dtype=np.int32), az


def _real_sh(l: int, m: int, theta: np.ndarray, phi: np.ndarray) -> np.ndarray:
    from scipy.special import sph_harm_y
    if m == 0:
        return np.real(sph_harm_y(l, 0, theta, phi))
    y = sph_harm_y(l, abs(m), theta, phi)
    return math.sqrt(2.0) * (-1) ** m * (np.real(y) if m > 0 else np.imag(y))


def sh_displace(verts: np.ndarray, rng: np.random.Generator, lmax: int = 4) -> np.ndarray:
    """Low-frequency seeded displacement r = 1 + sum_{l=1..4} c_lm Y_lm, c_lm ~ N(0,(0.1/l)^2),
    then scaled to max norm 1."""
    n = verts / np.linalg.norm(verts, axis=1, keepdims=True)
    theta = np.arccos(np.clip(n[:, 1], -1, 1))
    phi = np.arctan2(n[:, 2], n[:, 0])
    r = np.ones(len(verts))
    for l in range(1, lmax + 1):
        for m in range(-l, l + 1):
            r += rng.normal(0.0, 0.1 / l) * _real_sh(l, m, theta, phi)
    out = n * r[:, None]
    return out / np.max(np.linalg.norm(out, axis=1))


def rot_x(angle: float) -> np.ndarray:
    c, s = math.cos(angle), math.sin(angle)
    return np.array([[1, 0, 0], [0, c, -s], [0, s, c]])


def init_object(verts: np.ndarray, rng: np.random.Generator) -> np.ndarray:
    """Object initialisation: scale to max norm 1, then rotate about the
    local X axis by a uniform angle in [-90, 90] degrees."""
    v = verts / np.max(np.linalg.norm(verts, axis=1))
    return v @ rot_x(math.radians(rng.uniform(-90.0, 90.0))).T


# --------------------------------------------------------------------------- cameras / motion

def spherical_eye(d: float, elev_deg: float, azim_deg: float) -> np.ndarray:
    """y-up spherical placement (SURVEY Q5 reading of A33)."""
    p, t = math.radians(elev_deg), math.radians(azim_deg)
    return np.array([d * math.cos(p) * math.sin(t), d * math.sin(p), d * math.cos(p) * math.cos(t)])


def camera_row(eye, target=(0, 0, 0), up=(0, 1, 0), half_fov=HALF_FOV, z_near=Z_NEAR):
    return np.concatenate([np.asarray(eye, float), np.asarray(target, float),
                           np.asarray(up, float), [half_fov, z_near]]).astype(np.float32)


def motion_arrays(rows):
    """rows: list of dicts(kind, vec, angle, pivot, N, S, rule)."""
    B = len(rows)
    out = dict(kind=np.zeros(B, np.int32), vec=np.zeros((B, 3), np.float32),
               angle=np.zeros(B, np.float32), pivot=np.zeros((B, 3), np.float32),
               n_sub=np.zeros(B, np.int32), n_seg=np.zeros(B, np.int32), rule=np.zeros(B, np.int32))
    for b, r in enumerate(rows):
        out["kind"][b] = r.get("kind", STATIC)
        out["vec"][b] = r.get("vec", (0, 0, 0))
        out["angle"][b] = r.get("angle", 0.0)
        out["pivot"][b] = r.get("pivot", (0, 0, 0))
        out["n_sub"][b] = r["N"]
        out["n_seg"][b] = r.get("S", 1)
        out["rule"][b] = r.get("rule", GLOBAL_INCLUSIVE)
    return out


def translate(T, N, S=1, rule=GLOBAL_INCLUSIVE):
    """P(t) = P0 + (t - 0.5) T  (A30 generalised; the paper's case is T = (-1,0,0))."""
    return dict(kind=TRANSLATE, vec=T, N=N, S=S, rule=rule)


def rotate(axis, angle, N, S, pivot=(0, 0, 0), rule=GLOBAL_INCLUSIVE):
    """P(t) = c + R(axis, angle * t)(P0 - c)  (A31 generalised)."""
    a = np.asarray(axis, float)
    return dict(kind=ROTATE, vec=a / np.linalg.norm(a), angle=angle, pivot=pivot, N=N, S=S, rule=rule)


def parabolic(N, S, axis=(0, 1, 0), angle=math.pi, pivot=(0, 0, 0), rule=GLOBAL_INCLUSIVE):
    """A35-A37: rotation R(axis, angle t) then translation (s, -4s^2 + 0.5, s),
    s = 0.5 - t; the paper's case is axis y, angle pi."""
    a = np.asarray(axis, float)
    return dict(kind=PARABOLIC, vec=a / np.linalg.norm(a), angle=angle, pivot=pivot, N=N, S=S, rule=rule)


def exact_pose(motion: dict) -> dict:
    """The same motion sampled at its exact poses: N sub-frames on N-1 segments (GLOBAL_INCLUSIVE
    puts sub-frame k on the keyframe t = k/(N-1)), the segmentation-error reference of NEXT-3."""
    m = dict(motion)
    m["S"] = max(1, int(m["N"]) - 1)
    m["rule"] = GLOBAL_INCLUSIVE
    return m


def static(N=1, S=1, rule=GLOBAL_INCLUSIVE):
    return dict(kind=STATIC, N=N, S=S, rule=rule)


# --------------------------------------------------------------------------- configs

def _colors(rng, V):
    return rng.uniform(0.0, 1.0, size=(V, 3)).astype(np.float32)


def _targets(rng, B, H, W):
    return rng.uniform(0.0, 1.0, size=(B, H, W, 4)).astype(np.float32)


def make_c1(seed: int = MASTER_SEED + 0) -> Scene:
    rng = np.random.default_rng(seed)
    v, f = icosphere(1, 0.5)
    cams = np.stack([camera_row((0, 0, 3))])
    mo = motion_arrays([translate((1.5, 0, 0), N=8, S=1)])
    return Scene("C1", v.astype(np.float32), f, _colors(rng, len(v)), cams, mo, 64, 64,
                 _targets(rng, 1, 64, 64))


def make_c2(seed: int = MASTER_SEED + 1) -> Scene:
    rng = np.random.default_rng(seed)
    v, f = icosphere(3, 0.5)
    v = v + rng.normal(0.0, 0.02, size=v.shape)
    col = _colors(rng, len(v))
    d = rng.normal(size=3)
    d /= np.linalg.norm(d)
    cams = np.stack([camera_row(spherical_eye(3.0, 0.0, az)) for az in (0, 90, 180, 270)])
    mo = motion_arrays([translate(3.0 * d, N=50, S=1)] * 4)
    return Scene("C2", v.astype(np.float32), f, col, cams, mo, 256, 256, _targets(rng, 4, 256, 256))


def make_c3(seed: int = MASTER_SEED + 2) -> Scene:
    rng = np.random.default_rng(seed)
    v, f, az = revolution_top(rng)
    c = rng.uniform(0.0, 1.0, size=(2, 3))
    sector = (az * 8) // 80
    col = np.where((sector % 2 == 0)[:, None], c[0], c[1]).astype(np.float32)
    cams = np.stack([camera_row(spherical_eye(CAM_DIST, 30.0, a)) for a in range(0, 360, 45)])
    tilt = math.radians(20.0)
    axis = (math.sin(tilt), math.cos(tilt), 0.0)
    mo = motion_arrays([rotate(axis, 4 * math.pi, N=50, S=24)] * 8)
    return Scene("C3", v.astype(np.float32), f, col, cams, mo, 512, 512, _targets(rng, 8, 512, 512))


_TRANS_ELEV = (-60, -30, 0, 30, 60)
_TRANS_AZIM = (-315, -270, -225, -180, -135, -90, -45, 0)


def _inverse_step(name, level, n_views_each, res, N, seed, rot_elevs):
    rng = np.random.default_rng(seed)
    sphere, f = icosphere(level, 1.0)
    # the displaced mesh plays the role of the unknown object; the optimised mesh is the template
    # sphere.  Both get the paper's object initialisation.
    rot = math.radians(rng.uniform(-90.0, 90.0))
    displaced = sh_displace(sphere, rng) @ rot_x(rot).T
    template = sphere @ rot_x(rot).T
    col = _colors(rng, len(sphere))
    grid = [(e, a) for e in _TRANS_ELEV for a in _TRANS_AZIM]
    pick = rng.choice(len(grid), size=n_views_each, replace=False)
    cams, rows = [], []
    for i in sorted(pick):
        e, a = grid[i]
        cams.append(camera_row(spherical_eye(CAM_DIST, e, a)))
        rows.append(translate((-1.0, 0.0, 0.0), N=N, S=1))
    for e in rot_elevs:
        cams.append(camera_row(spherical_eye(CAM_DIST, e, 0.0)))
        rows.append(rotate((0, 1, 0), 2 * math.pi, N=N, S=12))
    B = len(cams)
    sc = Scene(name, template.astype(np.float32), f, col, np.stack(cams), motion_arrays(rows),
               res, res, _targets(rng, B, res, res))
    sc.meta["displaced_verts"] = displaced.astype(np.float32)
    return sc


def make_c4(seed: int = MASTER_SEED + 3) -> Scene:
    return _inverse_step("C4", 5, 8, 512, 100, seed, (-60, -45, -30, -15, 0, 15, 30, 60))


def make_c5(seed: int = MASTER_SEED + 4) -> Scene:
    return _inverse_step("C5", 6, 32, 1024, 256, seed, tuple(np.linspace(-60.0, 60.0, 32)))


CONFIGS = {"C1": make_c1, "C2": make_c2, "C3": make_c3, "C4": make_c4, "C5": make_c5}


def make(name: str) -> Scene:
    return CONFIGS[name]()


# --------------------------------------------------------------------------- tiny scenes for pins

def single_scene(verts, faces, colors, cam=None, motion=None, H=16, W=16, seed=0, B=1):
    rng = np.random.default_rng(seed)
    cam = camera_row((0, 0, 3)) if cam is None else cam
    motion = static(1) if motion is None else motion
    return Scene("tiny", np.asarray(verts, np.float32), np.asarray(faces, np.int32),
                 np.asarray(colors, np.float32), np.stack([cam] * B), motion_arrays([motion] * B),
                 H, W, _targets(rng, B, H, W))


def random_mesh_scene(n_faces: int, seed: int, H: int = 16, W: int = 16, motion=None, B: int = 1):
    """Tiny random triangle soup in front of a camera on +z (for brute-force pins)."""
    rng = np.random.default_rng(seed)
    V = 3 * n_faces
    centres = rng.uniform(-0.6, 0.6, size=(n_faces, 1, 3))
    verts = (centres + rng.normal(0, 0.35, size=(n_faces, 3, 3))).reshape(V, 3)
    faces = np.arange(V, dtype=np.int32).reshape(n_faces, 3)
    motion = translate((0.8, 0.3, 0.2), N=5) if motion is None else motion
    return single_scene(verts, faces, rng.uniform(0, 1, (V, 3)), motion=motion, H=H, W=W,
                        seed=seed + 1, B=B)


def cube(half: float = 0.5, centre=(0.0, 0.0, 0.0)):
    """Closed axis-aligned cube (8 V / 12 F, outward-facing), for the voxel-IoU pins."""
    c = np.asarray(centre, np.float64)
    v = np.array([[x, y, z] for x in (-half, half) for y in (-half, half) for z in (-half, half)]) + c
    f = [(0, 1, 3), (0, 3, 2), (4, 6, 7), (4, 7, 5), (0, 4, 5), (0, 5, 1),
         (2, 3, 7), (2, 7, 6), (0, 2, 6), (0, 6, 4), (1, 5, 7), (1, 7, 3)]
    return v, np.array(f, dtype=np.int32)


def star(k: int = 6, radius: float = 1.0):
    """Fan of k triangles around vertex 0 (ring vertices 1..k), for the Laplacian closed form."""
    ring = [[radius * math.cos(2 * math.pi * i / k), radius * math.sin(2 * math.pi * i / k), 0.0] for i in range(k)]
    v = np.array([[0.0, 0.0, 0.0]] + ring)
    f = [(0, 1 + i, 1 + (i + 1) % k) for i in range(k)]
    return v, np.array(f, dtype=np.int32)
