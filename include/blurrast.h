/*
 * blurrast.h -- C ABI of the B200 (sm_100a) motion-blur rasterizer: the hot path of
 * arxiv 2602.07860 ("fast barycentric coordinate solver", section 3).
 *
 * Citations: P:L### = line of the paper's LaTeX source; Eq.n numbered in
 * \begin{equation} order; A# = appendix equation; S:L### = SPEC.md; Q# = a reading of a
 * silent/ambiguous passage, listed in DESIGN.md.
 *
 * What one call computes: for B observed images of one triangle mesh under a
 * known rigid motion, the blurred RGBA image
 *     I_b(p) = (1/N) sum_k [ covered_k(p) ? (sum_i w_i(tau_k) c_i, 1) : (0,0,0,0) ]
 * where sub-frame k lies in segment s_k at segment time tau_k (Q1), the keyframes of segment s are
 * the exact rigid pose at t = s/S projected with A34, vertices move linearly in
 * screen space inside a segment (Eq.4-6), the barycentric weights are evaluated with
 * the paper's fast solver w(tau) = (A1 tau^2 + A2 tau + A3)/(a1 tau^2 + a2 tau + a3) (Eq.8,
 * P:L264; A11-A16) from coefficients computed once per (face, segment), a pixel is
 * covered by a face iff all w_i >= 0 (Q7), the nearest covering face by interpolated view
 * depth wins (Z-buffer, Q6; lower face index on exact ties), and shading is Eq.9
 * with background (0,0,0,0) (Q10).  blur_render_bwd scatters dL/dI into per-vertex
 * world-position and colour gradients through the same weights, frozen winners (Q11).
 *
 * Conventions for every entry point:
 *  - Pointers are DEVICE pointers unless the comment says "host".  The caller owns every buffer;
 *    the library keeps no allocation and no global state except a thread-local error string.
 *  - Work is enqueued asynchronously on `stream` (a cudaStream_t; 0 = legacy default stream).
 *    Argument errors are detected synchronously and returned before anything is enqueued.
 *    Data-dependent errors (face index >= V, a vertex behind the near plane, bin overflow) are
 *    recorded in a status word inside the workspace; read it with blur_read_status().  Faces with
 *    an invalid index or a vertex behind the near plane are skipped, never clipped.
 *    Bin overflow is not an error for the result: the affected tiles take a slower exact path.
 *  - Layouts: verts [V,3] f32 world positions; faces [F,3] i32; colors [V,3] f32; images
 *    [B,H,W,4] f32 RGBA, row 0 at the top, pixel (i,j) centre at NDC
 *    (-1 + (2i+1)/W, 1 - (2j+1)/H) (Q9).
 *  - Return value: a blur_status.  blur_last_error() gives a message for the last non-OK return
 *    on the calling thread.
 *  - Re-entrant on distinct workspaces/streams.  Setting BLURRAST_CHECK=1 in the environment makes
 *    every render call synchronise and return the device status word.
 */
#ifndef BLURRAST_H
#define BLURRAST_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *blur_stream_t; /* == cudaStream_t */

typedef enum {
    BLUR_OK = 0,
    BLUR_EINVAL = 1,    /* invalid argument (sync) or face index out of range (status word) */
    BLUR_EBEHIND = 2,   /* a vertex at or behind the near plane at some keyframe (status word) */
    BLUR_ENOMEM = 3,    /* workspace smaller than blur_workspace_bytes() */
    BLUR_ECUDA = 4,     /* a CUDA launch or copy failed */
    BLUR_EOVERFLOW = 5  /* bin capacity exceeded: result exact, some tiles took the slow path */
} blur_status;

/* status-word bits (blur_read_status) */
#define BLUR_ST_EINVAL 1
#define BLUR_ST_EBEHIND 2
#define BLUR_ST_EOVERFLOW 4
#define BLUR_ST_EINTERNAL 8   /* internal consistency check failed (a bug: please report) */

typedef enum { BLUR_STATIC = 0, BLUR_TRANSLATE = 1, BLUR_ROTATE = 2, BLUR_PARABOLIC = 3 } blur_motion_kind;
typedef enum { BLUR_SCHED_GLOBAL_INCLUSIVE = 0, BLUR_SCHED_PAPER_SEGMENTED = 1 } blur_sched_rule;

/* Motion over the exposure t in [0,1] (host struct, one per image).
 *  BLUR_TRANSLATE: P(t) = P0 + (t - 0.5) vec          (A30, generalised; Q2)
 *  BLUR_ROTATE:    P(t) = c + R(vec, angle t)(P0 - c)  (A31, generalised; Q3, Q4:
 *                  right-handed Rodrigues rotation about the unit axis vec through c = pivot)
 *  BLUR_PARABOLIC: P(t) = c + R(vec, angle t)(P0 - c) + (s, -4 s^2 + 0.5, s), s = 0.5 - t
 *                  (composite rotation + parabolic translation, A35-A37; the paper's
 *                  case is vec = +y, angle = pi, c = 0).  Not linear in t: use several segments.
 *  n_subframes N >= 1; n_segments S >= 1 (linear segments), or 0 for the automatic
 *  count: 1 for translation / static, ceil(12 |angle| / 2 pi - 1e-6) for rotation / parabolic (12 per
 *  full turn; Q24); sched_rule as Q1:
 *   GLOBAL_INCLUSIVE: t_k = k/(N-1) (N=1: 0.5), s_k = min(floor(t_k S), S-1), tau_k = t_k S - s_k;
 *   PAPER_SEGMENTED:  S | N, K = N/S, s_k = k div K, tau_k = (k mod K)/(K-1) (K=1: 0.5). */
typedef struct {
    int32_t kind;
    float vec[3];
    float angle;
    float pivot[3];
    int32_t n_subframes;
    int32_t n_segments;
    int32_t sched_rule;
} blur_motion;

/* Pinhole camera (host struct, one per image): looks from eye at target; right = normalize(f x up),
 * up' = right x f; view coords Q = (right.(P-E), up'.(P-E), f.(P-E)); NDC x = Qx/(Qz tan(half_fov)),
 * y = Qy/(Qz tan(half_fov)) (A34; Q5).  A vertex with Qz <= z_near is invalid. */
typedef struct {
    float eye[3];
    float target[3];
    float up[3];
    float half_fov;   /* radians, in (0, pi/2) */
    float z_near;     /* > 0 */
} blur_camera;

/* Tuning / instrumentation (host struct; NULL = defaults). */
#define BLUR_REUSE_SETUP 1   /* bwd: reuse keyframes, coefficients and bins that the preceding fwd
                                call with identical arguments left in the same workspace */
#define BLUR_TABLES_RESIDENT 4   /* fwd: the workspace already holds the host-side tables (schedule,
                                poses, chunks) of a previous call with identical arguments; skip their
                                upload.  With it a fwd/bwd pair issues device work only, so it can be
                                captured in a CUDA graph and replayed (BlurRenderer.capture_step). */
#define BLUR_CACHE_VISIBILITY 2   /* set on both the fwd and the bwd call: the fwd also leaves the
                                winning bin slot of every (pixel, sub-frame) in the workspace (2 B each:
                                sum_b N_b * H * W * 2 bytes, e.g. 0.84 GB for C4), and a bwd with
                                BLUR_REUSE_SETUP reads it instead of recomputing the visibility (the
                                result is identical; solver 0 only).  An index buffer, not sub-frame
                                images: the blurred image is still accumulated in registers.  With
                                delta > 0 the soft forward (K8) also leaves, per background (pixel,
                                sub-frame), the product of the factors 1 - A_j (Eq.15; 4 B each) that
                                the soft backward (K9) needs for dalpha/dA_j, instead of recomputing
                                them. */
typedef struct {
    int32_t max_chunk;             /* G: max sub-frames sharing one tile bin (0 = automatic) */
    int32_t flags;                 /* BLUR_REUSE_SETUP */
    float bin_factor;              /* bin-entry capacity per (chunk, face) (0 = default 3.0); see
                                      blur_read_bins for sizing it to the geometry */
    unsigned long long *census;    /* device u64[12] or NULL: fwd adds [covered (pixel,face,subframe)
                                      pairs, covered (pixel,subframe), candidate pair tests,
                                      staged (face,subframe,tile) records (these four: every bin face
                                      tested at its footprints, the algorithmic counts), soft
                                      (pixel,face,subframe) terms evaluated, staged soft records, soft
                                      work items (sub-frame, 8x4 footprint), soft face iterations of
                                      those items, then the same first four counts for the timed
                                      fast-solver forward, which skips faces hidden behind nearer
                                      winners] (a census call renders the batch twice) */
    void *raster_events[2];        /* host cudaEvent_t pair or NULLs: recorded on `stream` right
                                      before / after the raster kernel (K4 in fwd, K6 in bwd), for
                                      timing the dominant kernel inside a step */
    int32_t solver;                /* barycentric solver (NEXT-2 ablation of P:L447-479):
                                      0 = fast (default): Eq.8 with the per-segment coefficients,
                                      1 = naive per-frame: lerp the keyframe vertices and set the
                                          triangle up again at every sub-frame (same per-pixel work),
                                      2 = naive per-pixel: re-solve w = F(tau)^-1 p (Eq.3) for every
                                          (pixel, face, sub-frame) test (the SoftRas-style baseline) */
    /* Soft background coverage (NEXT-1; Eq.10-15; A17-A20).  delta > 0
     * gives every pixel that no face covers at a sub-frame RGB 0 and alpha
     *   A_i(t) = 1 - prod_j (1 - exp(-d_j / delta)),  d_j = || p - F_j(tau) w^* ||^2  (Eq.15, Eq.10, Eq.14)
     * with w^* the closest point (A17-A18) of p' = F_j(X) w_j(tau) on the keyframe triangle
     * F_j(X), X = [tau > 0.5] (Eq.13); delta in NDC^2 (the paper's 1e-4; Q9).  The
     * backward then also carries dL/dalpha into the vertex gradients, w^* held constant.
     * Needs solver 0.  delta = 0: hard coverage only (alpha = coverage, the delta -> 0 limit). */
    float delta;
    float soft_cut;                /* faces with d > soft_cut * delta are dropped (their term is below
                                      exp(-soft_cut)); 0 = default 18: beyond it the forward's fp32
                                      factor 1 - A is exactly 1 (Q21) */
    int32_t soft_exact;            /* 1: Eq.12 (closest point on F(tau) itself) instead of Eq.13 */
    float soft_bin_factor;         /* soft-bin entry capacity per (chunk, face) (0 = default 12); see
                                      blur_read_soft_bins */
    void *soft_events[2];          /* host cudaEvent_t pair or NULLs: recorded around the soft kernel
                                      (K8 in fwd, K9 in bwd) */
} blur_config;

/* Bytes of device workspace the render calls need for these arguments (0 + blur_last_error() on
 * invalid arguments).  `motions`, `cams` and `sub_range` are host arrays as in blur_render_fwd. */
size_t blur_workspace_bytes(int V, int F, int B, int H, int W, const blur_motion *motions,
                            const blur_camera *cams, const int32_t *sub_range, const blur_config *cfg);

/* Forward: blurred images.
 *  verts [V,3], faces [F,3], colors [V,3]: device, read-only.
 *  motions [B], cams [B]: host.
 *  sub_range: host [B][2] half-open sub-frame ranges [k0,k1) per image, or NULL for [0,N).
 *  out_rgba [B,H,W,4]: overwritten with (1/N) sum over k in [k0,k1) of the sub-frame values, so
 *    partial ranges add up (sub-frame sharding).
 *  ids [B,H,W] or NULL: winning face index at sub-frame ids_subframe (-1 = background); pixels of
 *    images whose [k0,k1) does not contain ids_subframe are left untouched.
 *  ws / ws_bytes: device workspace of at least blur_workspace_bytes(...). */
int blur_render_fwd(const float *verts, int V, const int32_t *faces, int F, const float *colors,
                    const blur_motion *motions, const blur_camera *cams, int B, int H, int W,
                    const int32_t *sub_range, float *out_rgba, int32_t *ids, int ids_subframe,
                    const blur_config *cfg, void *ws, size_t ws_bytes, blur_stream_t stream);

/* Backward: grad_rgba [B,H,W,4] = dL/d out_rgba (device).  grad_verts [V,3] and grad_colors [V,3]
 * are OVERWRITTEN with dL/dverts (world) and dL/dcolors summed over the B images and the sub-frame
 * ranges.  The alpha channel carries no position gradient in the hard-coverage path; with
 * cfg->delta > 0 it does, through the soft background term (w^* frozen).
 * With cfg->flags & BLUR_REUSE_SETUP the setup stages of the preceding blur_render_fwd on the same
 * workspace with identical arguments are reused. */
int blur_render_bwd(const float *verts, int V, const int32_t *faces, int F, const float *colors,
                    const blur_motion *motions, const blur_camera *cams, int B, int H, int W,
                    const int32_t *sub_range, const float *grad_rgba, float *grad_verts,
                    float *grad_colors, const blur_config *cfg, void *ws, size_t ws_bytes,
                    blur_stream_t stream);

/* L2 image loss (BASELINE C1 "L2 loss"; Q14): loss[0] = sum((out - target)^2) / n_norm and
 * grad = 2 (out - target) / n_norm over n elements (n_norm <= 0 -> n).  loss is a device float,
 * overwritten; grad may alias nothing else. */
int blur_l2_loss_grad(const float *out, const float *target, int64_t n, int64_t n_norm, float *loss,
                      float *grad, blur_stream_t stream);

/* Synchronises `stream`, reads the status word of `ws` (BLUR_ST_* bits) into *status_out (host) and
 * clears it. */
int blur_read_status(void *ws, blur_stream_t stream, int32_t *status_out);

/* Synchronises `stream` and reports, for the last binning done in `ws`, the number of bin entries
 * the geometry needed (*needed, host) and the capacity the workspace had (*capacity, host).  When
 * needed > capacity the affected tiles took the exact slow path (BLUR_EOVERFLOW): size the next
 * workspace with cfg->bin_factor scaled by needed / capacity.  blur_read_soft_bins: the same for
 * the soft-coverage bins (cfg->soft_bin_factor; 0 / 0 when delta == 0). */
int blur_read_bins(void *ws, blur_stream_t stream, long long *needed, long long *capacity);
int blur_read_soft_bins(void *ws, blur_stream_t stream, long long *needed, long long *capacity);

/* FP32 FFMA throughput microbenchmark (roofline denominator): runs `iters` iterations of 8
 * independent FMA chains per thread on ctas x 256 threads; writes 2 * flops-per-launch into
 * *flops (host) and sinks results into sink (device, >= ctas*256 floats). */
int blur_ffma_probe(int ctas, int iters, float *sink, double *flops, blur_stream_t stream);

/* Message for the last non-OK return on this thread ("" if none). */
const char *blur_last_error(void);

/* ABI version (increments on incompatible change). */
int blur_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* BLURRAST_H */
