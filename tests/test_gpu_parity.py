"""GPU parity: the CUDA path (through the C ABI) vs the fp64 CPU oracle on the same seeded inputs.

Bars (BASELINE.json north_star; readings Q16/Q18 in DESIGN.md):
  * visible-triangle-ID map bit-exact except at (pixel, sub-frame) the oracle flags as ambiguous
    (within 1e-6 NDC of an edge or a 1e-6 relative depth tie, Q16);
  * blurred intensities within 1e-4 max-abs on non-ambiguous pixels;
  * vertex gradients (dV and dC separately) within 1e-3 relative L2, same upstream G on both sides.
"""
import numpy as np
import pytest

import oracle
import scenes

pytestmark = pytest.mark.gpu

TOL_IMG = 1e-4
TOL_GRAD = 1e-3


def _torch():
    import torch
    return torch


def gpu_render(sc, ids_k=-1, sub_range=None, max_chunk=0, bin_factor=0.0, G=None, reuse=True, cache=False):
    torch = _torch()
    from paper_2602_07860_b200 import BlurRenderer
    dev = torch.device("cuda:0")
    r = BlurRenderer(sc.faces, sc.motion, sc.cams, sc.H, sc.W, sc.V, device=dev, sub_range=sub_range,
                     max_chunk=max_chunk, bin_factor=bin_factor, cache_visibility=cache)
    v = torch.tensor(np.asarray(sc.verts, np.float32), device=dev)
    c = torch.tensor(np.asarray(sc.colors, np.float32), device=dev)
    ids = torch.full((sc.B, sc.H, sc.W), -7, dtype=torch.int32, device=dev) if ids_k >= 0 else None
    out = r.forward(v, c, ids=ids, ids_subframe=ids_k)
    res = dict(rgba=out.cpu().numpy(), ids=None if ids is None else ids.cpu().numpy())
    if G is not None:
        g = torch.tensor(np.asarray(G, np.float32), device=dev)
        dv, dc = r.backward(v, c, g, reuse_setup=reuse)
        res["dv"], res["dc"] = dv.cpu().numpy(), dc.cpu().numpy()
    torch.cuda.synchronize()
    res["status"] = r.status()
    return res


def rel_l2(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


# Caps on the excluded fractions of the touched pixels (alpha > 0 in the oracle); a mask that grows past
# them hides real mismatches.  eps is fixed in NDC (1e-6), i.e. wider in pixels at higher resolution, so
# the share of pixel centres within eps of an edge in one sub-frame grows linearly with W; amb_win takes
# the union over the N sub-frames, so it grows with N as well.  Measured: amb_img 0.04-0.08% on C2-C4 at
# 512^2 and below, 0.15% on C5 (1024^2); amb_win 0.25% (C2, N = 50, 256^2), 1.6-2.4% (C4, N = 100, 512^2),
# 9.2% (C5, N = 256, 1024^2).
def mask_caps(W, N):
    s = max(1.0, W / 512.0)
    return 1e-3 * s, 3e-4 * N * s      # C4: 0.1% and 3%; C5: 0.2% and 15%


def mask_fractions(ref, N, min_touched=2000):
    """Excluded fractions of the touched pixels; asserts the caps when the image has enough touched
    pixels for a fraction to mean something."""
    touched = ref["rgba"][..., 3] > 0
    nt = max(int(touched.sum()), 1)
    f_img, f_win = float((ref["amb_img"] & touched).sum()) / nt, float((ref["amb_win"] & touched).sum()) / nt
    cap_img, cap_win = mask_caps(ref["rgba"].shape[2], N)
    print("excluded of %d touched pixels: amb_img %.3f%% (cap %.2f%%) amb_win %.3f%% (cap %.2f%%)"
          % (nt, 100 * f_img, 100 * cap_img, 100 * f_win, 100 * cap_win))
    if nt >= min_touched:
        assert f_img <= cap_img, "amb_img excludes %.3f%% of the touched pixels" % (100 * f_img)
        assert f_win <= cap_win, "amb_win excludes %.3f%% of the touched pixels" % (100 * f_win)
    return dict(touched=nt, amb_img_frac=f_img, amb_win_frac=f_win)


def check_parity(sc, ids_k=0, mode="binned", max_chunk=0, sub_range=None, grad=True, all_pixel_grad=True,
                 gpu_sc=None, views=None, cache=False):
    """Oracle vs GPU on sc.  gpu_sc/views: the GPU renders gpu_sc (e.g. the whole batch in the bench's
    launch configuration) and its images `views` are compared with sc (= gpu_sc.subset(views))."""
    ref = oracle.render_fwd(sc, mode=mode, ids_k=ids_k, eps_amb=1e-6, sub_range=sub_range)
    out = mask_fractions(ref, int(max(sc.motion["n_sub"])))
    # the same upstream G on both sides (the oracle's image), zero where the winner of some
    # sub-frame is ambiguous: the frozen-winner derivative is discontinuous there (Q18)
    G_all = 2.0 * (ref["rgba"] - sc.target) / ref["rgba"].size if grad else None
    G = G_all * (~ref["amb_win"])[..., None] if grad else None

    def embed(Gs):
        if gpu_sc is None or Gs is None:
            return Gs
        Gb = np.zeros((gpu_sc.B, gpu_sc.H, gpu_sc.W, 4), np.float32)
        Gb[views] = Gs
        return Gb

    got = gpu_render(gpu_sc or sc, ids_k=ids_k, sub_range=sub_range, max_chunk=max_chunk, G=embed(G), cache=cache)
    if gpu_sc is not None:
        got["rgba"], got["ids"] = got["rgba"][views], got["ids"][views]
    assert not (got["status"] & 8), "internal consistency check failed"
    ok = ~ref["amb_img"]
    err = np.abs(got["rgba"] - ref["rgba"])
    assert err[ok].max() < TOL_IMG, "image max err %g (all pixels %g)" % (err[ok].max(), err.max())
    okid = ~ref["amb_ids"]
    mism = (got["ids"] != ref["ids"]) & okid
    assert not mism.any(), "id mismatch at %d pixels" % mism.sum()
    out.update(img_err=float(err[ok].max()), img_err_all=float(err.max()), amb=int((~ok).sum()),
               amb_win=int(ref["amb_win"].sum()), pixels=int(ok.size),
               ids_equal_all=float((got["ids"] == ref["ids"]).mean()))
    if grad:
        rdv, rdc = oracle.render_bwd(sc, G, mode=mode, sub_range=sub_range)
        ev, ec = rel_l2(got["dv"], rdv), rel_l2(got["dc"], rdc)
        assert ev < TOL_GRAD and ec < TOL_GRAD, "grad rel L2 dV %g dC %g" % (ev, ec)
        out.update(dv=ev, dc=ec)
        if all_pixel_grad:   # reported beside the excluded one: the same comparison with G unmasked
            adv, adc = oracle.render_bwd(sc, G_all, mode=mode, sub_range=sub_range)
            ga = gpu_render(gpu_sc or sc, sub_range=sub_range, max_chunk=max_chunk, G=embed(G_all), cache=cache)
            out.update(dv_all_pixels=rel_l2(ga["dv"], adv), dc_all_pixels=rel_l2(ga["dc"], adc))
    return out


def test_large_image_global_binning_path():
    """Images with more than 4096 tiles take K3's global-atomic count/fill (the shared-histogram
    variants need the tile counters in shared memory): 1100 x 1040 pixels = 69 x 65 tiles."""
    sc = scenes.random_mesh_scene(40, 17, H=1040, W=1100, motion=scenes.translate((0.6, -0.2, 0.1), N=3))
    r = check_parity(sc, ids_k=1)
    print(r)


def test_c1_full_brute():
    r = check_parity(scenes.make_c1(), ids_k=3, mode="brute")
    print(r)


def test_c2_full():
    r = check_parity(scenes.make_c2(), ids_k=17)
    print(r)


def test_c3_subset():
    r = check_parity(scenes.make_c3().subset([0, 3, 6]), ids_k=25)
    print(r)


def test_c3_full_batch():
    """C3 (BASELINE configs[2]): all 8 views, the rotating top, compared completely."""
    r = check_parity(scenes.make_c3(), ids_k=25)
    print(r)


def test_c4_full_batch_bench_path():
    """C4 (BASELINE configs[3], the bench workload): all 16 views in one launch with the visibility cache and
    the K6 gather, as bench.py times them, compared completely with the binned oracle."""
    r = check_parity(scenes.make_c4(), ids_k=40, cache=True)
    print(r)


def test_c4_two_views():
    sc = scenes.make_c4().subset([2, 11])   # one translational, one rotational view
    r = check_parity(sc, ids_k=40)
    print(r)


def test_c5_full_views_in_bench_launch():
    """C5 (BASELINE configs[4]: 64 x 1024^2, N = 256, 81,920 faces) rendered as the bench renders it
    (the whole 64-image batch in one launch: its bins take the long-bin and batched paths); one
    translational and one rotational view compared completely with the binned oracle."""
    full = scenes.make_c5()
    views = [0, 63]
    assert full.motion["kind"][0] != full.motion["kind"][63]
    r = check_parity(full.subset(views), ids_k=128, gpu_sc=full, views=views)
    print(r)


@pytest.mark.parametrize("k,x_c", [(0, 0.5), (2, -0.5)])
def test_translation_time_direction_gpu(k, x_c):
    """A30, x(t) = x0 + (0.5 - t): sub-frame k = 0 (t = 0) of the paper's translation
    T = (-1, 0, 0) shows the object at x0 + 0.5, sub-frame 2 (t = 1) at x0 - 0.5 (camera on the z axis,
    half field of view 45 deg: NDC x = world x; cf. tests/test_oracle_masks.py)."""
    import math
    half, hh, Wd = 0.1, 0.3, 40
    cam = scenes.camera_row((0, 0, 1), half_fov=math.pi / 4, z_near=0.05)
    verts = [(-half, -hh, 0), (half, -hh, 0), (half, hh, 0), (-half, hh, 0)]
    sc = scenes.single_scene(verts, [[0, 1, 2], [0, 2, 3]], np.full((4, 3), 0.5), cam=cam,
                             motion=scenes.translate((-1.0, 0, 0), N=3), H=8, W=Wd)
    a = gpu_render(sc, sub_range=[[k, k + 1]])["rgba"][0, ..., 3]
    us = -1 + (2 * np.arange(Wd) + 1) / Wd
    vs = 1 - (2 * np.arange(8) + 1) / 8
    inside = (np.abs(us[None, :] - x_c) < half - 1e-6) & (np.abs(vs[:, None]) < hh - 1e-6)
    outside = (np.abs(us[None, :] - x_c) > half + 1e-6) | (np.abs(vs[:, None]) > hh + 1e-6)
    assert inside.sum() >= 8
    assert np.allclose(a[inside], 1.0 / 3.0, atol=1e-7) and np.all(a[outside] == 0.0)


@pytest.mark.parametrize("G", [1, 3, 16])
def test_chunk_length_invariance(G):
    """The per-sub-frame result does not depend on the bin chunk length G: ID maps bit-identical;
    images equal up to the order of the fp32 sub-frame sum (small launches split the sub-frames
    over several CTAs, see K4)."""
    sc = scenes.make_c2().subset([0, 2])
    a = gpu_render(sc, ids_k=5, max_chunk=G)
    b = gpu_render(sc, ids_k=5, max_chunk=8)
    assert np.array_equal(a["ids"], b["ids"])
    assert np.abs(a["rgba"] - b["rgba"]).max() < 1e-6


def test_overflow_fallback_exact():
    """A tiny bin capacity forces the exact fallback path (faces rescanned in index order)."""
    sc = scenes.make_c2().subset([1])
    G = np.random.default_rng(0).normal(size=(1, 256, 256, 4)) * 1e-4
    a = gpu_render(sc, ids_k=7, G=G)
    b = gpu_render(sc, ids_k=7, bin_factor=1e-9, G=G)
    assert b["status"] & 4                     # BLUR_ST_EOVERFLOW reported
    assert np.array_equal(a["ids"], b["ids"]) and np.abs(a["rgba"] - b["rgba"]).max() < 1e-6
    assert rel_l2(b["dv"], a["dv"]) < 1e-5 and rel_l2(b["dc"], a["dc"]) < 1e-5


def test_sub_range_partials_sum_to_full():
    """Sub-frame sharding: renders over [0,k) and [k,N) add up to the full render."""
    sc = scenes.make_c3().subset([1, 5])
    full = gpu_render(sc)["rgba"]
    a = gpu_render(sc, sub_range=[[0, 20], [0, 33]])["rgba"]
    b = gpu_render(sc, sub_range=[[20, 50], [33, 50]])["rgba"]
    assert np.max(np.abs(a + b - full)) < 2e-6
    ref = oracle.render_fwd(sc, sub_range=[[0, 20], [0, 33]], eps_amb=1e-6)
    ok = ~ref["amb_img"]
    assert np.abs(a - ref["rgba"])[ok].max() < TOL_IMG


def test_ragged_image_and_degenerate_faces():
    """Image size not a multiple of the tile; degenerate and repeated-index faces are skipped."""
    sc = scenes.random_mesh_scene(40, 5, H=37, W=53, motion=scenes.rotate((0.2, 1, 0.3), 1.2, N=9, S=4))
    faces = sc.faces.copy()
    faces[3] = [7, 7, 8]                       # repeated index
    verts = sc.verts.copy()
    verts[faces[5, 1]] = verts[faces[5, 0]]    # zero-area face
    sc.faces, sc.verts = faces, verts
    r = check_parity(sc, ids_k=4, mode="brute")
    print(r)


def test_paper_segmented_schedule_and_static():
    sc = scenes.random_mesh_scene(30, 8, H=40, W=40,
                                  motion=scenes.rotate((0, 1, 0), 6.283185307, N=60, S=12, rule=1))
    check_parity(sc, ids_k=11, mode="brute")
    st = scenes.random_mesh_scene(30, 9, H=40, W=40, motion=scenes.static(1))
    check_parity(st, ids_k=0, mode="brute")
    one = scenes.random_mesh_scene(30, 9, H=40, W=40, motion=scenes.translate((0.4, 0, 0), N=1))
    check_parity(one, ids_k=0, mode="brute")


def test_behind_camera_and_bad_index_status():
    sc = scenes.random_mesh_scene(20, 10, H=24, W=24, motion=scenes.static(1))
    v = sc.verts.copy()
    v[0] = [0, 0, 3.5]                         # behind the camera at z = 3
    sc.verts = v
    res = gpu_render(sc, ids_k=0)
    assert res["status"] & 2                   # BLUR_ST_EBEHIND
    ref = oracle.render_fwd(sc, ids_k=0, eps_amb=1e-6)
    ok = ~ref["amb_img"]
    assert np.abs(res["rgba"] - ref["rgba"])[ok].max() < TOL_IMG
    f = sc.faces.copy()
    f[2] = [0, 1, 10 ** 6]
    sc.faces = f
    res = gpu_render(sc, ids_k=0)
    assert res["status"] & 1                   # BLUR_ST_EINVAL
    assert not np.any(res["ids"] == 2)


def test_empty_mesh_and_empty_batch():
    torch = _torch()
    from paper_2602_07860_b200 import BlurRenderer
    sc = scenes.single_scene(np.zeros((3, 3)), np.zeros((0, 3), np.int32), np.zeros((3, 3)), H=20, W=30)
    got = gpu_render(sc, ids_k=0)
    assert not got["rgba"].any() and np.all(got["ids"] == -1)
    r = BlurRenderer(np.zeros((0, 3), np.int32), scenes.motion_arrays([]), np.zeros((0, 11)), 8, 8, 3)
    out = r.forward(torch.zeros((3, 3), device="cuda"), torch.zeros((3, 3), device="cuda"))
    assert out.shape == (0, 8, 8, 4)


def test_determinism():
    sc = scenes.make_c2().subset([3])
    a = gpu_render(sc, ids_k=9)
    b = gpu_render(sc, ids_k=9)
    assert np.array_equal(a["rgba"], b["rgba"]) and np.array_equal(a["ids"], b["ids"])


def test_invalid_arguments_raise():
    torch = _torch()
    from paper_2602_07860_b200 import BlurError, BlurRenderer
    sc = scenes.make_c1()
    bad = {k: v.copy() for k, v in sc.motion.items()}
    bad["n_sub"][0] = 0
    with pytest.raises(BlurError):
        BlurRenderer(sc.faces, bad, sc.cams, 64, 64, sc.V)
    cams = sc.cams.copy()
    cams[0, 9] = 2.0                            # half_fov >= pi/2
    with pytest.raises(BlurError):
        BlurRenderer(sc.faces, sc.motion, cams, 64, 64, sc.V)
    r = BlurRenderer(sc.faces, sc.motion, sc.cams, 64, 64, sc.V)
    with pytest.raises(TypeError):
        r.forward(torch.zeros((sc.V, 3), dtype=torch.float64, device="cuda"), torch.zeros((sc.V, 3), device="cuda"))


# ----------------------------------------------------------------- full-size (bench configuration)

def _sample_pixels(rng, B, H, W, n):
    b = rng.integers(0, B, n)
    j = rng.integers(H // 6, 5 * H // 6, n)
    i = rng.integers(W // 6, 5 * W // 6, n)
    return np.stack([b, j, i], 1).astype(np.int32)


@pytest.mark.parametrize("name,npix", [("C4", 96), ("C5", 24)])
def test_full_size_sampled(name, npix):
    """BASELINE full sizes in the launch configuration bench.py times (whole batch, automatic chunk
    length): sampled pixels computed one by one by the oracle (brute force over all faces and all
    sub-frames); gradients of a loss supported on the sampled pixels only (exact for the oracle)."""
    sc = scenes.make(name)
    rng = np.random.default_rng(123)
    pix = _sample_pixels(rng, sc.B, sc.H, sc.W, npix)
    Gp = rng.normal(size=(npix, 4))
    G = np.zeros((sc.B, sc.H, sc.W, 4))
    G[pix[:, 0], pix[:, 1], pix[:, 2]] = Gp
    got = gpu_render(sc, ids_k=-1, G=G)
    ref = oracle.render_fwd(sc, pixels=pix, eps_amb=1e-6)
    g_img = got["rgba"][pix[:, 0], pix[:, 1], pix[:, 2]]
    ok = ~ref["amb_img"]
    assert ok.sum() >= npix * 0.8
    err = np.abs(g_img - ref["rgba"])[ok]
    assert err.max() < TOL_IMG, err.max()
    # the loss reads only the sampled pixels; winner-ambiguous ones are excluded on both sides (Q18)
    Gp2 = Gp * (~ref["amb_win"])[:, None]
    G2 = np.zeros_like(G)
    G2[pix[:, 0], pix[:, 1], pix[:, 2]] = Gp2
    got2 = gpu_render(sc, G=G2)
    rdv, rdc = oracle.render_bwd(sc, Gp2, pixels=pix)
    assert rel_l2(got2["dv"], rdv) < TOL_GRAD and rel_l2(got2["dc"], rdc) < TOL_GRAD


# ----------------------------------------------------------------- NEXT-3: parabolic motion, exact-pose reference

def test_parabolic_motion_parity():
    sc = scenes.make_c2().subset([0, 1])
    sc.motion = scenes.motion_arrays([scenes.parabolic(N=40, S=8)] * 2)
    r = check_parity(sc, ids_k=13)
    print(r)


def test_exact_pose_reference_parity():
    sc = scenes.make_c3().subset([2])
    sc.motion = scenes.motion_arrays([scenes.exact_pose(scenes.rotate((0, 1, 0), 6.283185307, N=30, S=1))])
    r = check_parity(sc, ids_k=7)
    print(r)


# ----------------------------------------------------------------- NEXT-2: naive solvers (ablation baselines)

@pytest.mark.parametrize("solver", [1, 2])
def test_naive_solvers_match_oracle(solver):
    """The ablation baselines compute the same images/gradients (per-frame set-up, per-pixel solve)."""
    torch = _torch()
    from paper_2602_07860_b200 import BlurRenderer
    sc = scenes.make_c2().subset([0])
    ref = oracle.render_fwd(sc, eps_amb=1e-6)
    r = BlurRenderer(sc.faces, sc.motion, sc.cams, sc.H, sc.W, sc.V, solver=solver)
    out = r.forward(torch.tensor(sc.verts, device="cuda"), torch.tensor(sc.colors, device="cuda")).cpu().numpy()
    ok = ~ref["amb_img"]
    assert np.abs(out - ref["rgba"])[ok].max() < TOL_IMG
    G = 2.0 * (ref["rgba"] - sc.target) / ref["rgba"].size * (~ref["amb_win"])[..., None]
    dv, dc = r.backward(torch.tensor(sc.verts, device="cuda"), torch.tensor(sc.colors, device="cuda"),
                        torch.tensor(G, dtype=torch.float32, device="cuda"), reuse_setup=True)
    rdv, rdc = oracle.render_bwd(sc, G)
    assert rel_l2(dv.cpu().numpy(), rdv) < TOL_GRAD and rel_l2(dc.cpu().numpy(), rdc) < TOL_GRAD


@pytest.mark.parametrize("cfg", ["C2", "C3"])
def test_visibility_cache_equals_recompute(cfg):
    """BLUR_CACHE_VISIBILITY (K6 reads K4's winner slots, float moments) gives the same image and
    gradients as recomputing the visibility in K6 (k6_raster_bwd_fx: fixed-point moments, one rounding of
    2^-20 of the tile's largest |g| per pixel, amplified by the closed form's cancellation for faces far
    from the tile centre: ~1e-4 relative) and as a backward without the preceding forward."""
    sc = scenes.make(cfg).subset([0, 1])
    G = np.random.default_rng(3).normal(size=(sc.B, sc.H, sc.W, 4)).astype(np.float32) * 1e-4
    a = gpu_render(sc, G=G, cache=True)
    b = gpu_render(sc, G=G, cache=False)
    c = gpu_render(sc, G=G, cache=True, reuse=False)
    assert np.array_equal(a["rgba"], b["rgba"])
    for x in (b, c):
        ev, ec = rel_l2(x["dv"], a["dv"]), rel_l2(x["dc"], a["dc"])
        print(cfg, "dV %.2e dC %.2e" % (ev, ec))
        assert ev < 3e-4 and ec < 3e-4


def test_exact_depth_ties_lower_face_index_wins():
    """Q7: coincident faces (duplicated vertices, different colours) tie exactly in depth at every
    covered pixel; the lower face index must win, whatever order the (unsorted) bins visit them in."""
    rng = np.random.default_rng(8)
    base = scenes.random_mesh_scene(12, 21, H=40, W=40, motion=scenes.translate((0.5, 0.1, 0.0), N=6))
    V = base.V
    verts = np.concatenate([base.verts, base.verts]).astype(np.float32)
    cols = np.concatenate([base.colors, rng.uniform(0, 1, base.colors.shape)]).astype(np.float32)
    # interleave: the duplicate (second vertex copy) of face i gets index 2i, the original 2i + 1
    faces = np.empty((2 * base.F, 3), np.int32)
    faces[0::2] = base.faces + V
    faces[1::2] = base.faces
    sc = scenes.single_scene(verts, faces, cols, motion=scenes.translate((0.5, 0.1, 0.0), N=6), H=40, W=40)
    r = check_parity(sc, ids_k=2, mode="brute")
    got = gpu_render(sc, ids_k=2)
    ids = got["ids"][0]
    assert np.all((ids < 0) | (ids % 2 == 0))      # only the lower-index copies are visible
    print(r)


@pytest.mark.parametrize("cfg", ["C1", "C2"])
def test_cuda_graph_step_matches_eager(cfg):
    """BlurRenderer.capture_step: the replayed CUDA graph (fwd -> L2 -> bwd, tables resident) gives
    the eager step's loss, image and gradients, and follows in-place updates of the vertices."""
    import torch
    from paper_2602_07860_b200 import BlurRenderer
    sc = scenes.make(cfg)
    dev = torch.device("cuda:0")
    r = BlurRenderer(sc.faces, sc.motion, sc.cams, sc.H, sc.W, sc.V, device=dev)
    v = torch.tensor(sc.verts, device=dev)
    c = torch.tensor(sc.colors, device=dev)
    tgt = torch.tensor(sc.target, device=dev)
    sg = r.capture_step(v, c, tgt)
    for shift in (0.0, 0.01):
        v.copy_(torch.tensor(sc.verts, device=dev) + shift)
        loss, dv, dc, out = sg.replay()
        torch.cuda.synchronize()
        r2 = BlurRenderer(sc.faces, sc.motion, sc.cams, sc.H, sc.W, sc.V, device=dev)
        l2, dv2, dc2, out2 = r2.step(v.clone(), c, tgt)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy(), out2.cpu().numpy())
        # the L2 loss sums the CTAs' partials with float atomics: its last bits depend on their order
        assert abs(float(loss) - float(l2)) <= 1e-5 * abs(float(l2))
        assert rel_l2(dv.cpu().numpy(), dv2.cpu().numpy()) < 1e-5
        assert rel_l2(dc.cpu().numpy(), dc2.cpu().numpy()) < 1e-5


def test_automatic_segment_count_parity():
    """n_segments = 0 (Q24) resolves to the same segmentation on the GPU as in the oracle."""
    sc = scenes.random_mesh_scene(20, 31, H=40, W=40, motion=scenes.rotate((0.1, 1, 0.2), 3.0, N=13, S=0))
    r = check_parity(sc, ids_k=6, mode="brute")
    print(r)


def _orientation_scene(open_bowl: bool):
    """Scenes against the lean forward's visiting order (faces turned away from the camera -- by the sign of
    the mesh's signed volume -- are tested last, and skipped per footprint when every pixel already has a
    nearer winner): (a) an outward sphere with a smaller *inward*-wound sphere in front of it, so the faces
    nearest the camera are classified as turned away; (b) an open hemispherical bowl seen from inside, whose
    visible faces are turned away while its volume sign is arbitrary."""
    v1, f1 = scenes.icosphere(2, 0.5)
    if open_bowl:
        keep = [i for i, f in enumerate(f1) if v1[f].mean(0)[2] < 0.05]      # the half away from the camera
        v, f = v1, f1[keep]
    else:
        v2, f2 = scenes.icosphere(1, 0.22)
        v2 = v2 + np.array([0.05, 0.0, 0.75])
        v = np.concatenate([v1, v2])
        f = np.concatenate([f1, f2[:, ::-1] + len(v1)])                       # second sphere wound inward
    rng = np.random.default_rng(7 if open_bowl else 8)
    mo = scenes.translate((0.35, -0.15, 0.05), N=6)
    return scenes.single_scene(v, f.astype(np.int32), rng.uniform(0, 1, (len(v), 3)), motion=mo, H=96, W=96,
                               seed=9, B=2)


@pytest.mark.parametrize("open_bowl", [False, True])
def test_visiting_order_against_orientation(open_bowl):
    """The list-level skip of k4l_raster_fwd is exact whatever the orientation heuristic says: IDs, images and
    gradients match the oracle on meshes whose visible faces are the ones it tests last."""
    r = check_parity(_orientation_scene(open_bowl), ids_k=3)
    print(r)
