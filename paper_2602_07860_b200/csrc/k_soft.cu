// k_soft.cu -- NEXT-1: soft background coverage (Eq.10-15, A17-A20), K8 forward and K9 backward.
//
// A pixel that no face covers at sub-frame tau (background) gets RGB 0 and the alpha
//     A_i(t) = 1 - prod_j (1 - A_i^j(t)),   A_i^j(t) = exp(-d / delta)          (Eq.15, Eq.10, A20)
// with d from the paper's endpoint approximation: w(tau) from the fast solver (Eq.8), the point
// p' = F(X) w(tau) on the keyframe triangle X = [tau > 0.5] (Eq.13), its closest point on F(X) by
// the three-edge projection (A17-A18), mapped back with the same weights to F(tau) (Eq.14):
// d = || p - F(tau) w^* ||^2.  Faces farther than rcut = sqrt(soft_cut * delta) from the pixel at
// tau are dropped (their term is < exp(-soft_cut); Q21).
//
// Barycentric (Gram) form of A17-A18 (exact restatement): with E1 = v1 - v0,
// E2 = v2 - v0 of F(X) and sum w = 1, p' - v0 = w1 E1 + w2 E2, so every projection parameter is an
// affine function of (w1, w2):
//     t01 = w1 + w2 (E1.E2)/|E1|^2,   t12 = ((w1 - 1) E1.E12 + w2 E2.E12) / |E12|^2,
//     t20 = (1 - w2) - w1 (E1.E2)/|E2|^2,
// clamped to [0, 1], and the residual of candidate w^* is Delta = w - w^* (sum 0): p' - F(X) w^* =
// Delta1 E1 + Delta2 E2, and Eq.14's F(tau) w - F(tau) w^* = Delta1 E1(tau) + Delta2 E2(tau).  Per
// (pixel, face, tau) this is ~50 flops on (w1, w2) and four edge vectors.  (The residuals are
// formed as vectors, not as Gram quadratic forms: for sliver faces |Delta| reaches 1e3 and the
// quadratic form loses d to cancellation, found on C2.)
//
// Which (pixel, sub-frame) are background comes from the hard raster pass (K4), which leaves one
// coverage ballot per (sub-frame, tile, warp) in the workspace (1 bit per pixel and sub-frame).
// The soft kernels use their own bins (K3 on the chunk boxes grown by rcut, faces in index order).
//   K8 (fwd)  CTA = 16x16 tile.  Per group of sub-frames: every (face, tau) pair whose grown box
//             reaches the tile is staged once into an 80 B shared-memory record with a per-(tau,
//             8x4-footprint) bit mask of the footprints that need it (uncovered pixels within rcut
//             of the face at tau).  Work items (tau, footprint) with uncovered pixels are handed
//             to warps through a shared-memory queue (balances the very uneven silhouette tiles);
//             a warp's lanes are the footprint's pixels and fold their faces into prod (1 - A) in
//             face order; each pixel's thread then sums 1 - P over the group's sub-frames in order
//             (deterministic).
//   K9 (bwd)  w^* frozen: dalpha/dA_j = prod_{l != j} (1 - A_l), dA/dd = -A/delta,
//             dd/dv_i(tau) = -2 w^*_i (p - F(tau) w^*).  Per work item, pass 1 = K8's products (in
//             registers); pass 2 re-walks the item's faces, each lane forms its pixel's corner
//             gradient, a warp reduce-scatter (9 shuffles for 6 values) sums them over the footprint,
//             and 12 lanes add the (1 - tau, tau) keyframe split into the face slot's shared
//             accumulators, flushed with one vector RED per (corner, keyframe) per chunk.
#include <algorithm>
#include <cstdio>

#include "internal.cuh"
#include "../../include/blurrast.h"

namespace br {

namespace {

constexpr int SNW = NT / 32;     // warps per CTA
#ifndef BR_SOFT_CART
#define BR_SOFT_CART 1   // 1: closest points measured in Cartesian coordinates of F(X) (soft_eval)
#endif
#ifndef BR_SREC_F8
#define BR_SREC_F8 224
#endif
#ifndef BR_K8_MINB
#define BR_K8_MINB 6
#endif
#ifndef BR_K9C_MINB
#define BR_K9C_MINB 4      // K9C (cached products) CTAs per SM
#endif
#ifndef BR_K9_SPLIT
#define BR_K9_SPLIT 1
#endif
constexpr int SREC_F8 = BR_SREC_F8;   // K8: staged soft records per CTA (80 B each)
#ifndef BR_SREC_B9
#define BR_SREC_B9 384
#endif
#ifndef BR_K9_MINB
#define BR_K9_MINB 3
#endif
constexpr int SREC_B9 = BR_SREC_B9;   // K9: staged soft records per CTA
constexpr int GMAX_S = 8;        // sub-frames staged together
constexpr int NPX = TW * TH;

struct __align__(16) SoftRec {
    // q0: a1 b1 g1 a2 | q1: b2 g2 v0x r01 | q2: c1 c2 v0y r20 | q3: E1x E1y E2x E2y of F(X)
    // q4: E1x E1y E2x E2y of F(tau)
    //   w_i = a_i ul + b_i vl + g_i (i = 1, 2; fast solver at tau, tile-local pixel coordinates)
    //   t01 = sat(w1 + r01 w2), t12 = sat(c1 (w1 - 1) + c2 w2), t20 = sat((1 - w2) - r20 w1); a zero-length
    //   edge of F(X) has r = NaN, which sat() flushes to t = 0 (Q19); (v0x, v0y) = v0 of F(tau), tile-local
    float4 q[5];
};

struct STile {
    float uc, vc, sx, sy;
    int px0, py0, lxmax, lymax;
};

__device__ __forceinline__ void stile(const Tables &t, int tile, STile &tc)
{
    const int tx = tile % t.TX, ty = tile / t.TX;
    tc.px0 = tx * TW;
    tc.py0 = ty * TH;
    tc.lxmax = min(TW - 1, t.W - 1 - tc.px0);
    tc.lymax = min(TH - 1, t.H - 1 - tc.py0);
    const int ic = tc.px0 + TW / 2, jc = tc.py0 + TH / 2;
    tc.uc = (float)(-1.0 + (2.0 * ic + 1.0) / t.W);
    tc.vc = (float)(1.0 - (2.0 * jc + 1.0) / t.H);
    tc.sx = (float)(2.0 / t.W);
    tc.sy = (float)(2.0 / t.H);
}

__device__ __forceinline__ bool tile_range(float xmn, float xmx, float ymn, float ymx, int W, int H, const STile &tc,
                                           int &x0, int &x1, int &y0, int &y1)
{
    float a, b, c, d;
    ndc_to_index(xmn, xmx, W, false, a, b);
    ndc_to_index(ymn, ymx, H, true, c, d);
    a = fmaxf(a - tc.px0, 0.f);
    b = fminf(b - tc.px0, (float)tc.lxmax);
    c = fmaxf(c - tc.py0, 0.f);
    d = fminf(d - tc.py0, (float)tc.lymax);
    if (!(a <= b) || !(c <= d)) return false;
    x0 = (int)a; x1 = (int)b; y0 = (int)c; y1 = (int)d;
    return true;
}

// the per-tau box of a (face, segment) record grown by rcut, as a tile-local pixel range
__device__ __forceinline__ bool grown_box(const float4 *__restrict__ r, float tau, float rcut, int W, int H,
                                          const STile &tc, int &x0, int &x1, int &y0, int &y1)
{
    const float4 b0 = __ldg(r + 7), b1 = __ldg(r + 8);
    return tile_range(__fsub_rn(box_lerp(tau, b0.x, b1.x), rcut), __fadd_rn(box_lerp(tau, b0.y, b1.y), rcut),
                      __fsub_rn(box_lerp(tau, b0.z, b1.z), rcut), __fadd_rn(box_lerp(tau, b0.w, b1.w), rcut), W, H,
                      tc, x0, x1, y0, y1);
}

// Can any pixel centre of the local rect lie within rcut of the triangle (sign-normalised edge
// functions e_i = A_i ul + B_i vl + G_i, positive inside)?  False only if the rect lies more than
// rcut outside one edge line (then every point of it is farther than rcut from the triangle).
// thr_i = rcut |(A_i, B_i)| + rounding allowance (per record, bounded over the whole tile)
__device__ __forceinline__ bool rect_near(const float A[3], const float B[3], const float G[3], const float thr[3],
                                          int x0, int x1, int y0, int y1, const STile &tc)
{
    const float ulmin = (float)(x0 - TW / 2) * tc.sx, ulmax = (float)(x1 - TW / 2) * tc.sx;
    const float vlmin = (float)(TH / 2 - y1) * tc.sy, vlmax = (float)(TH / 2 - y0) * tc.sy;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const float m = G[i] + A[i] * (A[i] > 0.f ? ulmax : ulmin) + B[i] * (B[i] > 0.f ? vlmax : vlmin);
        if (m < -thr[i]) return false;
    }
    return true;
}

// Fallback batch builder: faces whose grown per-tau box overlaps the tile, in index order.
__device__ int soft_fallback_fill(const Tables &t, const float4 *__restrict__ rseg, float tau, const STile &tc,
                                  int cap, int &fpos, int *sid, int *swsum)
{
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int nb = 0;
    while (fpos < t.F) {
        const int f = fpos + tid;
        bool hit = false;
        if (f < t.F) {
            const float4 *r = rseg + (size_t)f * REC_F4;
            int x0, x1, y0, y1;
            hit = __float_as_int(__ldg(r + 6).w) >= 0 && grown_box(r, tau, t.rcut, t.W, t.H, tc, x0, x1, y0, y1);
        }
        const unsigned m = __ballot_sync(0xffffffffu, hit);
        if (lane == 0) swsum[warp] = __popc(m);
        __syncthreads();
        int pre = 0, tot = 0;
#pragma unroll
        for (int w = 0; w < SNW; ++w) {
            const int c = swsum[w];
            pre += w < warp ? c : 0;
            tot += c;
        }
        __syncthreads();
        if (nb + tot > cap) break;
        if (hit) sid[nb + pre + __popc(m & ((1u << lane) - 1u))] = f;
        nb += tot;
        fpos += NT;
    }
    __syncthreads();
    return nb;
}

struct SoftBin {
    const float4 *rseg, *key0, *key1;
    const int *ent;
    int n;
    bool fb;
};

__device__ __forceinline__ void soft_bin(const Tables &t, const ImgInfo &im, const Chunk &ch, int c, int tile,
                                         SoftBin &sb)
{
    const size_t bi = (size_t)c * t.T + tile;
    const long long o = t.sb.off[bi];
    sb.n = (int)(t.sb.off[bi + 1] - o);
    sb.fb = sb.n > t.sb.sortcap || o + sb.n > t.sb.cap;
    sb.ent = t.sb.entries + o;
    sb.rseg = t.rec + (size_t)(im.rec_off + (long long)ch.s * t.F) * REC_F4;
    sb.key0 = t.key + im.key_off + (size_t)ch.s * t.V;
    sb.key1 = sb.key0 + t.V;
}

// Stage one (face, tau) soft record for this tile.  need[w] = uncovered-pixel bits of footprint w
// at tau.  Returns the mask of footprints the record must visit (0 = none).
__device__ __forceinline__ uint32_t soft_stage(const Tables &t, const float4 *__restrict__ r,
                                               const float4 *__restrict__ key0, const float4 *__restrict__ key1,
                                               int f, float tau, const STile &tc, const uint32_t *need,
                                               float rcut, SoftRec &out)
{
    const float4 q6 = __ldg(r + 6);
    if (__float_as_int(q6.w) < 0) return 0u;                             // skipped face
    const float D = __fmaf_rn(tau, __fmaf_rn(tau, q6.x, q6.y), q6.z);   // det F(tau) (Eq.8 a-coefficients)
    if (!(fabsf(D) > EPS_D)) return 0u;                                 // Q8
    int x0, x1, y0, y1;
    if (!grown_box(r, tau, rcut, t.W, t.H, tc, x0, x1, y0, y1)) return 0u;
    const float sg = D < 0.f ? -1.f : 1.f;
    float A[3], B[3], G[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {   // Eq.8 numerators at tau, re-centred at the tile centre
        const float4 e0 = __ldg(r + 2 * i), e1 = __ldg(r + 2 * i + 1);   // ox oy a0 a1 | b0 b1 dax day
        float al, be, gp;
        rec_edge_at(e0, e1, tau, tc.uc, tc.vc, al, be, gp);
        A[i] = al * sg;
        B[i] = be * sg;
        G[i] = gp * sg;
    }
    float thr[3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
        thr[i] = rcut * sqrtf(A[i] * A[i] + B[i] * B[i]) +
                 1e-5f * (fabsf(A[i]) * (8.f * tc.sx) + fabsf(B[i]) * (8.f * tc.sy) + fabsf(G[i])) + 1e-30f;
    uint32_t fm = 0u;
    for (int wy = y0 >> 2; wy <= (y1 >> 2); ++wy)
        for (int wx = x0 >> 3; wx <= (x1 >> 3); ++wx) {
            const int w = wy * 2 + wx;
            if (!need[w]) continue;
            const int rx0 = max(x0, wx * 8), rx1 = min(x1, wx * 8 + 7);
            const int ry0 = max(y0, wy * 4), ry1 = min(y1, wy * 4 + 3);
            if (rect_near(A, B, G, thr, rx0, rx1, ry0, ry1, tc)) fm |= 1u << w;
        }
    if (!fm) return 0u;
    const float invD = 1.0f / fabsf(D);
    const float4 vc = __ldg(t.fcol + 3 * (size_t)f + 2);
    const int vid[3] = {__float_as_int(vc.y), __float_as_int(vc.z), __float_as_int(vc.w)};
    float xT[3], yT[3], xX[3], yX[3];
    const bool useX1 = tau > 0.5f;                                      // Eq.13: X = 1 iff tau > 0.5
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const float4 a = __ldg(key0 + vid[i]), b = __ldg(key1 + vid[i]);
        xT[i] = __fmaf_rn(tau, __fsub_rn(b.x, a.x), a.x);              // F(tau), Eq.5-6
        yT[i] = __fmaf_rn(tau, __fsub_rn(b.y, a.y), a.y);
        xX[i] = t.soft_exact ? xT[i] : (useX1 ? b.x : a.x);            // Eq.12 (exact) / Eq.13
        yX[i] = t.soft_exact ? yT[i] : (useX1 ? b.y : a.y);
    }
    // F(X): edge vectors, Gram entries and the projection coefficients (zero-length edge: t = 0, Q19)
    const float e1x = xX[1] - xX[0], e1y = yX[1] - yX[0], e2x = xX[2] - xX[0], e2y = yX[2] - yX[0];
    const float e3x = xX[2] - xX[1], e3y = yX[2] - yX[1];
    const float g11 = e1x * e1x + e1y * e1y, g22 = e2x * e2x + e2y * e2y, g12 = e1x * e2x + e1y * e2y;
    const float l12 = e3x * e3x + e3y * e3y;
    const float r01 = g11 > 0.f ? g12 / g11 : __int_as_float(0x7fffffff);
    const float r20 = g22 > 0.f ? g12 / g22 : __int_as_float(0x7fffffff);
    const float c1 = l12 > 0.f ? (e1x * e3x + e1y * e3y) / l12 : 0.f;
    const float c2 = l12 > 0.f ? (e2x * e3x + e2y * e3y) / l12 : 0.f;
#if BR_SOFT_CART
    // Cartesian form: p' - v0(X) = (p - v0(tau)) + w1 M1 + w2 M2 with M_i = E_i(X) - E_i(tau) (= 0 when tau is the
    // keyframe X), the closest point of each edge of F(X) by its projection parameter (A17), distances in F(X)
    (void)r01; (void)r20; (void)c1; (void)c2;
    const float f1x = xT[1] - xT[0], f1y = yT[1] - yT[0], f2x = xT[2] - xT[0], f2y = yT[2] - yT[0];   // F(tau)
    out.q[0] = make_float4(A[1] * invD, B[1] * invD, G[1] * invD, A[2] * invD);
    out.q[1] = make_float4(B[2] * invD, G[2] * invD, __fsub_rn(xT[0], tc.uc), __fsub_rn(yT[0], tc.vc));
    out.q[2] = make_float4(e1x, e1y, e2x, e2y);
    out.q[3] = make_float4(e1x - f1x, e1y - f1y, e2x - f2x, e2y - f2y);
    out.q[4] = make_float4(g11 > 0.f ? 1.0f / g11 : __int_as_float(0x7fffffff), g22 > 0.f ? 1.0f / g22 : __int_as_float(0x7fffffff),
                           l12 > 0.f ? 1.0f / l12 : __int_as_float(0x7fffffff), 0.f);
#else
    out.q[0] = make_float4(A[1] * invD, B[1] * invD, G[1] * invD, A[2] * invD);
    out.q[1] = make_float4(B[2] * invD, G[2] * invD, __fsub_rn(xT[0], tc.uc), r01);
    out.q[2] = make_float4(c1, c2, __fsub_rn(yT[0], tc.vc), r20);
    out.q[3] = make_float4(e1x, e1y, e2x, e2y);
    out.q[4] = make_float4(xT[1] - xT[0], yT[1] - yT[0], xT[2] - xT[0], yT[2] - yT[0]);   // F(tau)
#endif
    return fm;
}

// A = exp(-d / delta) (Eq.10, A20) as 2^(d kexp) with kexp = -log2(e) / delta, flushing results below
// 2^-126 to 0 (d > 87 delta, far past the cut-off): one multiply and one MUFU.EX2
__device__ __forceinline__ float soft_kexp(float delta) { return -1.4426950408889634f / delta; }
__device__ __forceinline__ float soft_A(float d, float kexp)
{
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(d * kexp));
    return y;
}

// One (pixel, face, tau) term: d (Eq.14), the chosen edge e (corners e, (e+1)%3) with parameter t,
// and the residual r = p - F(tau) w^* (Eq.14's vector).
struct SoftHit {
    float d, t, rx, ry;
    int e;
};

// || d1 E1 + d2 E2 ||^2
__device__ __forceinline__ float resid2(float d1, float d2, const float4 &E)
{
    const float rx = __fmaf_rn(d1, E.x, d2 * E.z), ry = __fmaf_rn(d1, E.y, d2 * E.w);
    return __fmaf_rn(rx, rx, ry * ry);
}

#if BR_SOFT_CART
// Cartesian closest point (A17-A18) of p' on F(X): p' is formed about v0 as (p - v0(tau)) + w1 M1 + w2 M2, so it
// is p itself when tau is the keyframe X, and each edge candidate's squared distance is measured directly.  (The
// barycentric form below measures them through w = F(tau)^-1 p; for a limb sliver -- det F ~ 5e-8 NDC^2 on C5 --
// w reaches ~1e4, the three edges' candidates lie within 1e-5 NDC of each other and their distances differ by
// ~5e-4 relative, below that form's fp32 resolution: a C5 view chose another edge than the oracle at tau = 0.)
__device__ __forceinline__ SoftHit soft_eval(const SoftRec &r, float ul, float vl)
{
    const float4 q0 = r.q[0], q1 = r.q[1], q2 = r.q[2], q3 = r.q[3], q4 = r.q[4];
    const float w1 = __fmaf_rn(q0.x, ul, __fmaf_rn(q0.y, vl, q0.z));   // w(tau), Eq.8
    const float w2 = __fmaf_rn(q0.w, ul, __fmaf_rn(q1.x, vl, q1.y));
    const float px = __fsub_rn(ul, q1.z), py = __fsub_rn(vl, q1.w);     // p - v0(tau)
    const float sx = __fmaf_rn(w1, q3.x, __fmaf_rn(w2, q3.z, px));     // p' - v0(X)
    const float sy = __fmaf_rn(w1, q3.y, __fmaf_rn(w2, q3.w, py));
    SoftHit h;
    // edge v0v1: w^* = (1 - t, t, 0), point t E1
    float tt = __saturatef(__fmaf_rn(sx, q2.x, sy * q2.y) * q4.x);
    float dx = __fmaf_rn(-tt, q2.x, sx), dy = __fmaf_rn(-tt, q2.y, sy);
    float best = __fmaf_rn(dx, dx, dy * dy);
    h.t = tt; h.e = 0;
    // edge v1v2: w^* = (0, 1 - t, t), point E1 + t (E2 - E1)
    const float e3x = q2.z - q2.x, e3y = q2.w - q2.y;
    const float ox = sx - q2.x, oy = sy - q2.y;
    tt = __saturatef(__fmaf_rn(ox, e3x, oy * e3y) * q4.z);
    dx = __fmaf_rn(-tt, e3x, ox); dy = __fmaf_rn(-tt, e3y, oy);
    float qq = __fmaf_rn(dx, dx, dy * dy);
    if (qq < best) { best = qq; h.t = tt; h.e = 1; }
    // edge v2v0: w^* = (t, 0, 1 - t), point E2 - t E2 (parameter from v2, as A17: a zero-length edge is v2, Q19)
    const float o2x = sx - q2.z, o2y = sy - q2.w;
    tt = __saturatef(-__fmaf_rn(o2x, q2.z, o2y * q2.w) * q4.y);
    dx = __fmaf_rn(tt, q2.z, o2x); dy = __fmaf_rn(tt, q2.w, o2y);
    qq = __fmaf_rn(dx, dx, dy * dy);
    if (qq < best) { h.t = tt; h.e = 2; }
    // Eq.14: d = || p - F(tau) w^* ||^2 with F(tau) = F(X) - M
    const float ws1 = h.e == 0 ? h.t : (h.e == 1 ? 1.f - h.t : 0.f);
    const float ws2 = h.e == 0 ? 0.f : (h.e == 1 ? h.t : 1.f - h.t);
    const float f1x = q2.x - q3.x, f1y = q2.y - q3.y, f2x = q2.z - q3.z, f2y = q2.w - q3.w;
    h.rx = px - __fmaf_rn(ws1, f1x, ws2 * f2x);
    h.ry = py - __fmaf_rn(ws1, f1y, ws2 * f2y);
    h.d = __fmaf_rn(h.rx, h.rx, h.ry * h.ry);
    return h;
}
#else
__device__ __forceinline__ SoftHit soft_eval(const SoftRec &r, float ul, float vl)
{
    const float4 q0 = r.q[0], q1 = r.q[1], q2 = r.q[2], q3 = r.q[3];
    const float w1 = __fmaf_rn(q0.x, ul, __fmaf_rn(q0.y, vl, q0.z));   // w(tau), Eq.8
    const float w2 = __fmaf_rn(q0.w, ul, __fmaf_rn(q1.x, vl, q1.y));
    SoftHit h;
    // the closest point of p' = F(X) w on F(X) (A17-A18): residual Delta = w - w^* in the (E1, E2) basis
    // edge v0v1: w^* = (1 - t, t, 0)
    float tt = __saturatef(__fmaf_rn(w2, q1.w, w1));
    float best = resid2(w1 - tt, w2, q3);
    h.t = tt; h.e = 0;
    // edge v1v2: w^* = (0, 1 - t, t)
    const float w1m = w1 - 1.f;
    tt = __saturatef(__fmaf_rn(w1m, q2.x, w2 * q2.y));
    float qq = resid2(w1m + tt, w2 - tt, q3);
    if (qq < best) { best = qq; h.t = tt; h.e = 1; }
    // edge v2v0: w^* = (t, 0, 1 - t)
    const float w2m = w2 - 1.f;
    tt = __saturatef(__fmaf_rn(-w1, q2.w, -w2m));
    qq = resid2(w1, w2m + tt, q3);
    if (qq < best) { h.t = tt; h.e = 2; }
    // Eq.14: d = || p - F(tau) w^* ||^2, formed from the pixel itself (F(tau) Delta equals it, but for a
    // far pixel of a sliver face w is ill-conditioned and F(tau) w no longer reproduces p in fp32)
    const float4 q4 = r.q[4];
    const float ws1 = h.e == 0 ? h.t : (h.e == 1 ? 1.f - h.t : 0.f);
    const float ws2 = h.e == 0 ? 0.f : (h.e == 1 ? h.t : 1.f - h.t);
    h.rx = __fsub_rn(ul, q1.z) - __fmaf_rn(ws1, q4.x, ws2 * q4.z);
    h.ry = __fsub_rn(vl, q2.z) - __fmaf_rn(ws1, q4.y, ws2 * q4.w);
    h.d = __fmaf_rn(h.rx, h.rx, h.ry * h.ry);
    return h;
}
#endif

// Stage faces [base, base + nb) of the bin (or sid[] in fallback mode) at the ng sub-frames taus:
// records rec[l * nb + j], masks wm[(l * SNW + w) * nw + j / 32] (cleared by the caller).
template <bool CENSUS>
__device__ __forceinline__ void soft_stage_group(const Tables &t, const SoftBin &sb, int nb, int base, const float *taus,
                                                 int ng, const STile &tc, const uint32_t (*need)[SNW], const int *sid,
                                                 SoftRec *rec, uint32_t *wm, unsigned long long &nstage, float rcut)
{
    const int nw = (nb + 31) >> 5;
    const float inv_ng = 1.0f / (float)ng;
    for (int p = threadIdx.x; p < nb * ng; p += NT) {
        const int j = div_small(p, inv_ng), l = p - j * ng;
        uint32_t any = 0u;
#pragma unroll
        for (int w = 0; w < SNW; ++w) any |= need[l][w];
        if (!any) continue;
        const int f = sb.fb ? sid[j] : __ldg(sb.ent + base + j);
        if ((unsigned)f >= (unsigned)t.F) {
            atomicOr(t.status, BLUR_ST_EINTERNAL);
            continue;
        }
        const uint32_t fm = soft_stage(t, sb.rseg + (size_t)f * REC_F4, sb.key0, sb.key1, f, taus[l], tc, need[l],
                                       rcut, rec[l * nb + j]);
        if (CENSUS) nstage += fm != 0u;
        const uint32_t bit = 0x80000000u >> (j & 31);
        for (uint32_t m = fm; m; m &= m - 1) atomicOr(wm + (l * SNW + (__ffs(m) - 1)) * nw + (j >> 5), bit);
    }
}

// prod over the masked faces of (1 - A) for one pixel (face order), with the product of the
// non-zero factors and the count of zero factors (for dalpha/dA in the backward)
template <bool CENSUS>
__device__ __forceinline__ void soft_product(const SoftRec *rec, const uint32_t *wm, int nw, float ul, float vl,
                                             float kexp, float &P, float &Pnz, int &nz, unsigned long long &npair)
{
    // words by pointer with a countdown (keeps the bound from being re-derived per word)
    for (int left = nw; left > 0; --left, ++wm, rec += 32) {
        uint32_t m = *wm;
        while (m) {
            const int k = __clz(m);
            m ^= 0x80000000u >> k;
            const SoftHit h = soft_eval(rec[k], ul, vl);
            const float A = soft_A(h.d, kexp);                       // Eq.10 with the exp kernel (A20)
            const float fac = 1.0f - A;
            if (fac == 0.f) nz++;                                    // Eq.15, zero factors counted apart
            else Pnz *= fac;
            if (CENSUS) npair++;
        }
    }
    P = nz ? 0.f : Pnz;   // the full product (callers start from P = Pnz = 1, nz = 0): bit-identical
}

__device__ __forceinline__ void load_need(const Tables &t, const ImgInfo &im, int k, int tile, int warp, int lane,
                                          bool extra, uint32_t *dst)
{
    const uint32_t cov = t.covbits[cov_word(t, im, k, tile) + warp];
    const unsigned m = __ballot_sync(0xffffffffu, !((cov >> lane) & 1u) && extra);
    if (lane == 0) *dst = m;
}

// next work item (sub-frame l, footprint w) of the shared queue for this warp; -1 when drained
__device__ __forceinline__ int next_item(int *head, int nitems, int lane)
{
    int it = 0;
    if (lane == 0) it = atomicAdd(head, 1);
    it = __shfl_sync(0xffffffffu, it, 0);
    return it < nitems ? it : -1;
}

__device__ __forceinline__ void footprint_pixel(int w, int lane, const STile &tc, int &p, float &ul, float &vl)
{
    const int lx = (w & 1) * 8 + (lane & 7), ly = (w >> 1) * 4 + (lane >> 3);
    p = ly * TW + lx;
    ul = (float)(lx - TW / 2) * tc.sx;
    vl = (float)(TH / 2 - ly) * tc.sy;
}

struct SoftFwdSmem {
    SoftRec rec[SREC_F8];
    uint32_t wm[GMAX_S * SNW * (SREC_F8 / 32 + 1)];
    uint32_t need[GMAX_S][SNW];
    float om[GMAX_S][NPX];     // 1 - P per (sub-frame of the group, pixel); P across batches
    int sid[SREC_F8];
    float taus[GMAX_S];
    int wsum[SNW];
    int head;
};

template <bool CENSUS>
__global__ void __launch_bounds__(NT, BR_K8_MINB) k8_soft_fwd(Tables t, unsigned long long *census)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SoftFwdSmem &S = *reinterpret_cast<SoftFwdSmem *>(smem_raw);
    const int b = blockIdx.y, tile = blockIdx.x;
    const ImgInfo &im = t.imgs[b];
    STile tc;
    stile(t, tile, tc);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int lx = (warp & 1) * 8 + (lane & 7), ly = (warp >> 1) * 4 + (lane >> 3);
    const int px = tc.px0 + lx, py = tc.py0 + ly, myp = ly * TW + lx;
    const bool inimg = px < t.W && py < t.H;
    const float kexp = soft_kexp(t.delta);
    float alpha = 0.f;
    unsigned long long npair = 0, nstage = 0, nitem = 0, nface = 0;

    for (int c = im.chunk_begin + (int)blockIdx.z; c < im.chunk_end; c += t.ssplits) {
        const Chunk ch = t.chunks[c];
        SoftBin sb;
        soft_bin(t, im, ch, c, tile, sb);
        if (sb.n == 0) continue;   // no face within rcut of the tile during the chunk: every P = 1
        if (!sb.fb && sb.n <= SREC_F8) {
            const int n = sb.n, Gs = min(GMAX_S, group_div(SREC_F8, n)), nw = (n + 31) >> 5;
            for (int kg = ch.k0; kg < ch.k1; kg += Gs) {
                const int ng = min(Gs, ch.k1 - kg);
                for (int l = 0; l < ng; ++l) load_need(t, im, kg + l, tile, warp, lane, inimg, &S.need[l][warp]);
                for (int i = threadIdx.x; i < ng * SNW * nw; i += NT) S.wm[i] = 0u;
                if (threadIdx.x < ng) S.taus[threadIdx.x] = t.sched_tau[im.sched_off + kg + threadIdx.x];
                if (threadIdx.x == 0) S.head = 0;
                __syncthreads();
                soft_stage_group<CENSUS>(t, sb, n, 0, S.taus, ng, tc, S.need, S.sid, S.rec, S.wm, nstage, t.rcut_f);
                __syncthreads();
                for (int it = next_item(&S.head, ng * SNW, lane), nx = 0; it >= 0; it = nx) {   // next item prefetched
                    nx = next_item(&S.head, ng * SNW, lane);
                    const int l = it / SNW, w = it - l * SNW;
                    if (CENSUS && lane == 0 && S.need[l][w]) {   // work items and their face iterations
                        nitem++;
                        for (int wd = 0; wd < nw; ++wd) nface += __popc(S.wm[(l * SNW + w) * nw + wd]);
                    }
                    if ((S.need[l][w] >> lane) & 1u) {
                        int p;
                        float ul, vl, P = 1.f, Pnz = 1.f;
                        int nz = 0;
                        footprint_pixel(w, lane, tc, p, ul, vl);
                        soft_product<CENSUS>(S.rec + l * n, S.wm + (l * SNW + w) * nw, nw, ul, vl, kexp, P, Pnz, nz,
                                             npair);
                        S.om[l][p] = 1.f - P;
                        if (t.spz)   // the backward's dalpha/dA factors (K9 skips its product pass)
                            t.spz[((size_t)(im.cov_off + kg + l) * t.T + tile) * NPX + p] =
                                nz == 0 ? Pnz : (nz == 1 ? -Pnz : __int_as_float(0x7fffffff));
                    }
                }
                __syncthreads();
                for (int l = 0; l < ng; ++l)                     // this pixel's sub-frames, in order
                    if ((S.need[l][warp] >> lane) & 1u) alpha += S.om[l][myp];
                __syncthreads();
            }
        } else {
            for (int k = ch.k0; k < ch.k1; ++k) {
                load_need(t, im, k, tile, warp, lane, inimg, &S.need[0][warp]);
                if (threadIdx.x == 0) S.taus[0] = t.sched_tau[im.sched_off + k];
                S.om[0][myp] = 1.f;
                S.om[1][myp] = 1.f;                                   // prod of the non-zero factors
                reinterpret_cast<int *>(S.om[2])[myp] = 0;           // zero factors
                __syncthreads();
                uint32_t anyn = 0u;
#pragma unroll
                for (int w = 0; w < SNW; ++w) anyn |= S.need[0][w];
                int base = 0, fpos = 0;
                while (anyn) {
                    const int nb = sb.fb ? soft_fallback_fill(t, sb.rseg, S.taus[0], tc, SREC_F8, fpos, S.sid, S.wsum)
                                         : (base < sb.n ? min(SREC_F8, sb.n - base) : 0);
                    if (nb == 0) break;
                    const int nw = (nb + 31) >> 5;
                    for (int i = threadIdx.x; i < SNW * nw; i += NT) S.wm[i] = 0u;
                    if (threadIdx.x == 0) S.head = 0;
                    __syncthreads();
                    soft_stage_group<CENSUS>(t, sb, nb, base, S.taus, 1, tc, S.need, S.sid, S.rec, S.wm, nstage, t.rcut_f);
                    __syncthreads();
                    // items (footprint, part of the words): a long bin gives one footprint's warp a
                    // whole batch otherwise; the parts' products (om rows 3.., sign / NaN = one / more
                    // zero factors) are folded into the pixel's running product in part order
                    const int LP = min(GMAX_S - 3, nw);
                    for (int it = next_item(&S.head, SNW * LP, lane), nx = 0; it >= 0; it = nx) {   // next item prefetched
                        nx = next_item(&S.head, SNW * LP, lane);
                        const int part = it % LP, w = it / LP;
                        if ((S.need[0][w] >> lane) & 1u) {
                            int p;
                            float ul, vl, P = 1.f, Pnz = 1.f;
                            int nz = 0;
                            footprint_pixel(w, lane, tc, p, ul, vl);
                            const int wd0 = part * nw / LP, wd1 = (part + 1) * nw / LP;
                            soft_product<CENSUS>(S.rec + (wd0 << 5), S.wm + w * nw + wd0, wd1 - wd0, ul, vl, kexp, P, Pnz,
                                                 nz, npair);
                            S.om[3 + part][p] = nz == 0 ? Pnz : (nz == 1 ? -Pnz : __int_as_float(0x7fffffff));
                        }
                    }
                    __syncthreads();
                    if ((S.need[0][warp] >> lane) & 1u) {
                        float pnz = S.om[1][myp];
                        int nz = reinterpret_cast<const int *>(S.om[2])[myp];
                        for (int part = 0; part < LP; ++part) {
                            const float e = S.om[3 + part][myp];
                            const unsigned u = __float_as_uint(e);
                            nz += (u & 0x7fffffffu) > 0x7f800000u ? 2 : (int)(u >> 31);
                            pnz *= fabsf(e);
                        }
                        nz = min(nz, 2);
                        S.om[1][myp] = pnz;
                        reinterpret_cast<int *>(S.om[2])[myp] = nz;
                        S.om[0][myp] = nz ? 0.f : pnz;
                    }
                    base += nb;
                    __syncthreads();
                }
                if ((S.need[0][warp] >> lane) & 1u) {
                    alpha += 1.f - S.om[0][myp];
                    if (t.spz) {   // the backward's dalpha/dA factors, as in the grouped path
                        const int nz = reinterpret_cast<const int *>(S.om[2])[myp];
                        const float pnz = S.om[1][myp];
                        t.spz[((size_t)(im.cov_off + k) * t.T + tile) * NPX + myp] =
                            nz == 0 ? pnz : (nz == 1 ? -pnz : __int_as_float(0x7fffffff));
                    }
                }
                __syncthreads();
            }
        }
    }
    if (inimg) t.spart[(size_t)blockIdx.z * ((size_t)t.B * t.H * t.W) + ((size_t)b * t.H + py) * t.W + px] =
        alpha / (float)im.N;
    if (CENSUS) {
        atomicAdd(census + 4, npair);
        atomicAdd(census + 5, nstage);
        atomicAdd(census + 6, nitem);
        atomicAdd(census + 7, nface);
    }
}

// out alpha += sum over splits of the soft partials (fixed order: deterministic)
__global__ void __launch_bounds__(256) k8_soft_reduce(const float *__restrict__ spart, float4 *__restrict__ out,
                                                      size_t n, int splits)
{
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        float a = spart[i];
        for (int z = 1; z < splits; ++z) a += spart[(size_t)z * n + i];
        out[i].w += a;
    }
}

// ------------------------------------------------------------------ backward

struct SoftBwdSmem {
    SoftRec rec[SREC_B9];
    uint32_t wm[GMAX_S * SNW * (SREC_B9 / 32 + 1)];
    uint32_t need[GMAX_S][SNW];
    float pnz[GMAX_S][NPX];
    unsigned short nz[GMAX_S][NPX];
    float ga[NPX];
    float acc[SREC_B9][12];    // per bin slot: d/d keyframe s (corners x, y), then keyframe s+1
    int sid[SREC_B9];
    float taus[GMAX_S];
    int wsum[SNW];
    unsigned short items[SNW * (SREC_B9 / 32)];   // long path: non-empty items w << 4 | batch
    int head, head2, nitems;
};

__device__ __forceinline__ void soft_flush(const Tables &t, const ImgInfo &im, int s, int f, const float *a)
{
    const float4 q = __ldg(t.fcol + 3 * (size_t)f + 2);
    const int vid[3] = {__float_as_int(q.y), __float_as_int(q.z), __float_as_int(q.w)};
    float2 *d0 = t.dkey + im.key_off + (size_t)s * t.V;
    float2 *d1 = d0 + t.V;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        if (a[2 * i] != 0.f || a[2 * i + 1] != 0.f) atomicAdd(d0 + vid[i], make_float2(a[2 * i], a[2 * i + 1]));
        if (a[6 + 2 * i] != 0.f || a[7 + 2 * i] != 0.f) atomicAdd(d1 + vid[i], make_float2(a[6 + 2 * i], a[7 + 2 * i]));
    }
}

// flush and clear the slot accumulators [0, nb)
template <class Sm>
__device__ __forceinline__ void flush_slots(Sm &S, const Tables &t, const ImgInfo &im, int s, int nb,
                                            const int *fid_of)
{
    for (int j = threadIdx.x; j < nb; j += NT) {
        float a[12];
        bool nzf = false;
#pragma unroll
        for (int i = 0; i < 12; ++i) { a[i] = S.acc[j][i]; nzf |= a[i] != 0.f; S.acc[j][i] = 0.f; }
        if (nzf) soft_flush(t, im, s, fid_of[j], a);
    }
}

// Pass 2 of one work item (sub-frame l, footprint w): for each masked face, every needing lane
// forms its pixel's corner gradient; the warp reduce-scatters the 6 values (8 with padding: 9
// shuffles) and the lanes holding the sums add the keyframe split into the slot accumulators.
// FUSED: the products come from a pass over the same faces in this call (the whole bin is staged);
// otherwise from S.pnz / S.nz (accumulated over the batches of a long bin).
template <bool FUSED>
__device__ __forceinline__ void soft_grad_item(SoftBwdSmem &S, const SoftRec *rec, const uint32_t *wm, int nw,
                                               int l, int w, int lane, const STile &tc, float kexp, float c2,
                                               int wd0 = 0, int wd1 = -1)
{
    if (wd1 < 0) wd1 = nw;
    const bool mine = (S.need[l][w] >> lane) & 1u;
    int p;
    float ul, vl;
    footprint_pixel(w, lane, tc, p, ul, vl);
    float pz = 0.f;
    int z = 2;
    if (mine) {
        if (FUSED) {   // pass 1 of this footprint: the products, in face order, kept in registers
            float P = 1.f;
            unsigned long long dummy = 0;
            pz = 1.f;
            z = 0;
            soft_product<false>(rec, wm, nw, ul, vl, kexp, P, pz, z, dummy);
            z = min(z, 2);
        } else {
            pz = S.pnz[l][p];
            z = S.nz[l][p];
        }
    }
    const float ga = mine ? S.ga[p] : 0.f;
    const float tau = S.taus[l];
    // lane owning reduced value vi after the reduce-scatter: vi = 4 b4 + 2 b3 + b2 (lanes with b1 = b0 = 0)
    const int vi = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
    for (int wd = wd0; wd < wd1; ++wd) {
        uint32_t m = wm[wd];
        while (m) {
            const int k = __clz(m);
            m ^= 0x80000000u >> k;
            const int j = (wd << 5) + k;
            float v[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) v[i] = 0.f;
            bool any = false;
            if (mine && z < 2) {
                const SoftRec &r = rec[j];
                const SoftHit h = soft_eval(r, ul, vl);
                const float A = soft_A(h.d, kexp);
                const float fac = 1.0f - A;
                const float dadA = z == 0 ? pz / fac : (fac == 0.f ? pz : 0.f);
                // dL/dv_i(tau) = G_a dalpha/dA (A / delta) 2 w^*_i (p - F(tau) w^*)
                const float cc = ga * dadA * A * c2;
                if (cc != 0.f) {
                    const float gx = cc * h.rx;
                    const float gy = cc * h.ry;
                    const int ia = h.e, ib = h.e == 2 ? 0 : h.e + 1;
                    const float wa = 1.f - h.t, wb = h.t;
#pragma unroll
                    for (int q = 0; q < 3; ++q) {
                        const float wq = (q == ia ? wa : 0.f) + (q == ib ? wb : 0.f);
                        v[2 * q] = wq * gx;
                        v[2 * q + 1] = wq * gy;
                    }
                    any = true;
                }
            }
            if (!__any_sync(0xffffffffu, any)) continue;
            // reduce-scatter 8 -> 4 -> 2 -> 1 values, then a 4-lane all-reduce
            const bool u16 = lane & 16, u8 = lane & 8, u4 = lane & 4;
            float k4[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float keep = u16 ? v[4 + i] : v[i], send = u16 ? v[i] : v[4 + i];
                k4[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
            }
            float k2[2];
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const float keep = u8 ? k4[2 + i] : k4[i], send = u8 ? k4[i] : k4[2 + i];
                k2[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
            }
            float s1;
            {
                const float keep = u4 ? k2[1] : k2[0], send = u4 ? k2[0] : k2[1];
                s1 = keep + __shfl_xor_sync(0xffffffffu, send, 4);
            }
            s1 += __shfl_xor_sync(0xffffffffu, s1, 2);
            s1 += __shfl_xor_sync(0xffffffffu, s1, 1);
            // all four lanes of a group hold the sum: lane 4g adds keyframe s, lane 4g+1 keyframe s+1
            if ((lane & 2) == 0 && vi < 6 && s1 != 0.f) {
                const bool k1 = lane & 1;
                atomicAdd(&S.acc[j][(k1 ? 6 : 0) + vi], (k1 ? tau : 1.f - tau) * s1);
            }
        }
    }
}

// position (0..31) of the r-th (0-based) set bit of x, counted from the least significant bit
__device__ __forceinline__ int nth_set_bit(uint32_t x, int r)
{
    int pos = 0;
#pragma unroll
    for (int s = 16; s; s >>= 1) {
        const int c = __popc(x & ((1u << s) - 1u));
        if (r >= c) { r -= c; x >>= s; pos += s; }
    }
    return pos;
}

// Pass 2 with K8's cached products, transposed: the lanes are faces -- batch b of 32 of the faces
// in the item's mask, compacted -- with the record in registers, and loop over the footprint's
// pixels (their gradient factor and products broadcast by shuffles), so each lane sums its own
// face's corner gradients over the pixels in registers: no cross-lane reduction per (pixel, face)
// term, one set of shared atomics per (face, item).
template <class Sm>
__device__ __forceinline__ void soft_grad_faces(Sm &S, const SoftRec *rec, const uint32_t *wm, int nw,
                                                int b, int l, int w, int lane, const STile &tc, float kexp, float c2,
                                                const float *pzc)
{
    // compaction: inclusive scan of the words' face counts (nw <= 32)
    const uint32_t myw = lane < nw ? wm[lane] : 0u;
    int incl = __popc(myw);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    if ((b << 5) >= total) return;                                      // warp-uniform
    const int idx = (b << 5) + lane;
    const bool has = idx < total;
    int wi = 0;                                                         // word holding face idx
    for (int j = 0; j < nw; ++j) wi += __shfl_sync(0xffffffffu, incl, j) <= idx;
    const uint32_t wv = __shfl_sync(0xffffffffu, myw, wi & 31);
    const int ex = __shfl_sync(0xffffffffu, incl, wi & 31) - __popc(wv);
    const int slot = (wi << 5) + nth_set_bit(__brev(wv), idx - ex);    // bit 31 - k = slot 32 wi + k
    int p;
    float ulp, vlp;
    footprint_pixel(w, lane, tc, p, ulp, vlp);
    float cp = 0.f, ep = 0.f;
    bool ok = false;
    if ((S.need[l][w] >> lane) & 1u) {
        ep = pzc[p];                    // K8's encoding: |ep| the non-zero product, sign = one zero factor
        ok = (__float_as_uint(ep) & 0x7fffffffu) <= 0x7f800000u;   // NaN: two or more zero factors
        cp = S.ga[p] * c2;
    }
    unsigned act = __ballot_sync(0xffffffffu, ok && cp != 0.f);   // pixels with a non-zero factor
    SoftRec r;
    if (has) r = rec[slot];
    float g[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    while (act) {
        const int q = __ffs(act) - 1;
        act &= act - 1;
        const float ul = __shfl_sync(0xffffffffu, ulp, q), vl = __shfl_sync(0xffffffffu, vlp, q);
        const float cq = __shfl_sync(0xffffffffu, cp, q), eq = __shfl_sync(0xffffffffu, ep, q);
        if (!has) continue;
        const SoftHit h = soft_eval(r, ul, vl);
        const float A = soft_A(h.d, kexp);
        const float fac = 1.0f - A;
        // dalpha/dA_j = prod_{l != j} (1 - A_l): the non-zero product over fac_j (fac_j > 0 then), or with
        // one zero factor the product itself at that face
        const float pzq = fabsf(eq);
        float rf;
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rf) : "f"(fac));
        const float dadA = !signbit(eq) ? pzq * rf : (fac == 0.f ? pzq : 0.f);
        // dL/dv_i(tau) = G_a dalpha/dA (A / delta) 2 w^*_i (p - F(tau) w^*)
        const float cc = cq * dadA * A;
        const float gx = cc * h.rx;
        const float gy = cc * h.ry;
        const float wa = 1.f - h.t, wb = h.t;
        // corners (e, e + 1 mod 3) of the chosen edge get weights (1 - t, t)
        const float w0 = h.e == 0 ? wa : (h.e == 2 ? wb : 0.f);
        const float w1 = h.e == 1 ? wa : (h.e == 0 ? wb : 0.f);
        const float w2 = h.e == 2 ? wa : (h.e == 1 ? wb : 0.f);
        g[0] = __fmaf_rn(w0, gx, g[0]); g[1] = __fmaf_rn(w0, gy, g[1]);
        g[2] = __fmaf_rn(w1, gx, g[2]); g[3] = __fmaf_rn(w1, gy, g[3]);
        g[4] = __fmaf_rn(w2, gx, g[4]); g[5] = __fmaf_rn(w2, gy, g[5]);
    }
    if (has) {
        const float tau = S.taus[l];
        float *a = S.acc[slot];
#pragma unroll
        for (int i = 0; i < 6; ++i)
            if (g[i] != 0.f) {
                atomicAdd(a + i, (1.f - tau) * g[i]);   // keyframe s
                atomicAdd(a + 6 + i, tau * g[i]);       // keyframe s + 1
            }
    }
}

// bins K9C takes: K8 cached their products (grouped or per-sub-frame path) and K9C's record stage holds them
__device__ __forceinline__ bool k9c_bin(const SoftBin &sb) { return !sb.fb && sb.n <= SREC_B9; }

struct SoftBwdCSmem {
    SoftRec rec[SREC_B9];
    uint32_t wm[GMAX_S * SNW * (SREC_B9 / 32 + 1)];
    uint32_t need[GMAX_S][SNW];
    float ga[NPX];
    float acc[SREC_B9][12];    // per bin slot: d/d keyframe s (corners x, y), then keyframe s+1
    unsigned short items[GMAX_S * SNW * (SREC_B9 / 32)];   // non-empty work items: (l * SNW + w) << 4 | batch
    float taus[GMAX_S];
    int head2, nitems;
};

// K9C: the soft backward of the bins whose dalpha/dA products K8 left in t.spz (BLUR_CACHE_VISIBILITY):
// per group of sub-frames, stage the records, then work items (sub-frame, footprint, batch of 32
// faces) through soft_grad_faces.  Launched before K9, which takes every other bin.
__global__ void __launch_bounds__(NT, BR_K9C_MINB) k9c_soft_bwd(Tables t, const float *__restrict__ grad)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SoftBwdCSmem &S = *reinterpret_cast<SoftBwdCSmem *>(smem_raw);
    const int b = blockIdx.y, tile = blockIdx.x;
    const ImgInfo &im = t.imgs[b];
    STile tc;
    stile(t, tile, tc);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int lx = (warp & 1) * 8 + (lane & 7), ly = (warp >> 1) * 4 + (lane >> 3);
    const int px = tc.px0 + lx, py = tc.py0 + ly, myp = ly * TW + lx;
    const bool inimg = px < t.W && py < t.H;
    const float kexp = soft_kexp(t.delta), c2 = 2.0f / t.delta;
    const float ga = inimg ? __ldg(grad + 4 * (((size_t)b * t.H + py) * t.W + px) + 3) / (float)im.N : 0.f;
    S.ga[myp] = ga;
    const bool want = inimg && ga != 0.f;
    for (int i = threadIdx.x; i < SREC_B9 * 3; i += NT) reinterpret_cast<float4 *>(&S.acc[0][0])[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    unsigned long long dummy = 0;
    __syncthreads();

    for (int c = im.chunk_begin + (int)blockIdx.z; c < im.chunk_end; c += t.ssplits) {
        const Chunk ch = t.chunks[c];
        SoftBin sb;
        soft_bin(t, im, ch, c, tile, sb);
        if (sb.n == 0 || !k9c_bin(sb)) continue;
        const int n = sb.n, Gs = min(GMAX_S, group_div(SREC_B9, n)), nw = (n + 31) >> 5;
        bool touched = false;
        for (int kg = ch.k0; kg < ch.k1; kg += Gs) {
            const int ng = min(Gs, ch.k1 - kg);
            for (int l = 0; l < ng; ++l) load_need(t, im, kg + l, tile, warp, lane, want, &S.need[l][warp]);
            for (int i = threadIdx.x; i < ng * SNW * nw; i += NT) S.wm[i] = 0u;
            if (threadIdx.x < ng) S.taus[threadIdx.x] = t.sched_tau[im.sched_off + kg + threadIdx.x];
            if (threadIdx.x == 0) { S.head2 = 0; S.nitems = 0; }
            __syncthreads();
            uint32_t anyn = 0u;
            for (int l = 0; l < ng; ++l)
#pragma unroll
                for (int w = 0; w < SNW; ++w) anyn |= S.need[l][w];
            if (anyn) {   // block-uniform
                touched = true;
                soft_stage_group<false>(t, sb, n, 0, S.taus, ng, tc, S.need, nullptr, S.rec, S.wm, dummy, t.rcut);
                __syncthreads();
                // list the non-empty items (sub-frame, footprint, batch of 32 masked faces)
                for (int lw = warp; lw < ng * SNW; lw += SNW) {
                    if (!S.need[0][lw]) continue;   // need[l][w] == need[0][lw]
                    const unsigned cnt = lane < nw ? __popc(S.wm[lw * nw + lane]) : 0u;
                    const int nb = (int)((__reduce_add_sync(0xffffffffu, cnt) + 31u) >> 5);
                    int base = 0;
                    if (lane == 0 && nb) base = atomicAdd(&S.nitems, nb);
                    base = __shfl_sync(0xffffffffu, base, 0);
                    if (lane < nb) S.items[base + lane] = (unsigned short)((lw << 4) | lane);
                }
                __syncthreads();
                const int nit = S.nitems;
                for (int it = next_item(&S.head2, nit, lane), nx = 0; it >= 0; it = nx) {   // next item prefetched
                    nx = next_item(&S.head2, nit, lane);
                    const int v = S.items[it], lw = v >> 4, l = lw / SNW, w = lw - l * SNW;
                    soft_grad_faces(S, S.rec + l * n, S.wm + lw * nw, nw, v & 15, l, w, lane, tc, kexp, c2,
                                    t.spz + ((size_t)(im.cov_off + kg + l) * t.T + tile) * NPX);
                }
            }
            __syncthreads();
        }
        if (touched) {
            flush_slots(S, t, im, ch.s, n, sb.ent);
            __syncthreads();
        }
    }
}

__global__ void __launch_bounds__(NT, BR_K9_MINB) k9_soft_bwd(Tables t, const float *__restrict__ grad)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SoftBwdSmem &S = *reinterpret_cast<SoftBwdSmem *>(smem_raw);
    const int b = blockIdx.y, tile = blockIdx.x;
    const ImgInfo &im = t.imgs[b];
    STile tc;
    stile(t, tile, tc);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int lx = (warp & 1) * 8 + (lane & 7), ly = (warp >> 1) * 4 + (lane >> 3);
    const int px = tc.px0 + lx, py = tc.py0 + ly, myp = ly * TW + lx;
    const bool inimg = px < t.W && py < t.H;
    const float kexp = soft_kexp(t.delta), c2 = 2.0f / t.delta;
    const float ga = inimg ? __ldg(grad + 4 * (((size_t)b * t.H + py) * t.W + px) + 3) / (float)im.N : 0.f;
    S.ga[myp] = ga;
    const bool want = inimg && ga != 0.f;
    for (int i = threadIdx.x; i < SREC_B9 * 3; i += NT) reinterpret_cast<float4 *>(&S.acc[0][0])[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    unsigned long long dummy = 0;
    __syncthreads();

    for (int c = im.chunk_begin + (int)blockIdx.z; c < im.chunk_end; c += t.ssplits) {
        const Chunk ch = t.chunks[c];
        SoftBin sb;
        soft_bin(t, im, ch, c, tile, sb);
        if (sb.n == 0 || (t.spz && k9c_bin(sb))) continue;   // empty, or K9C's
        if (!sb.fb && sb.n <= SREC_B9) {
            const int n = sb.n, Gs = min(GMAX_S, group_div(SREC_B9, n)), nw = (n + 31) >> 5;
            bool touched = false;
            for (int kg = ch.k0; kg < ch.k1; kg += Gs) {
                const int ng = min(Gs, ch.k1 - kg);
                for (int l = 0; l < ng; ++l) load_need(t, im, kg + l, tile, warp, lane, want, &S.need[l][warp]);
                for (int i = threadIdx.x; i < ng * SNW * nw; i += NT) S.wm[i] = 0u;
                if (threadIdx.x < ng) S.taus[threadIdx.x] = t.sched_tau[im.sched_off + kg + threadIdx.x];
                if (threadIdx.x == 0) { S.head = 0; S.head2 = 0; }
                __syncthreads();
                uint32_t anyn = 0u;
                for (int l = 0; l < ng; ++l)
#pragma unroll
                    for (int w = 0; w < SNW; ++w) anyn |= S.need[l][w];
                if (anyn) {   // block-uniform
                    touched = true;
                    soft_stage_group<false>(t, sb, n, 0, S.taus, ng, tc, S.need, S.sid, S.rec, S.wm, dummy, t.rcut);
                    __syncthreads();
#if BR_K9_SPLIT
                    for (int it = next_item(&S.head, ng * SNW, lane), nx = 0; it >= 0; it = nx) {   // next item prefetched
                        nx = next_item(&S.head, ng * SNW, lane);
                        const int l = it / SNW, w = it - l * SNW;
                        if ((S.need[l][w] >> lane) & 1u) {
                            int p;
                            float ul, vl, P = 1.f, Pnz = 1.f;
                            int nz = 0;
                            footprint_pixel(w, lane, tc, p, ul, vl);
                            soft_product<false>(S.rec + l * n, S.wm + (l * SNW + w) * nw, nw, ul, vl, kexp, P, Pnz, nz,
                                                dummy);
                            S.pnz[l][p] = Pnz;
                            S.nz[l][p] = (unsigned short)min(nz, 2);
                        }
                    }
                    __syncthreads();
                    // pass 2: finer items (sub-frame, footprint, 32-face word) keep the tail short
                    for (int it = next_item(&S.head2, ng * SNW * nw, lane), nx = 0; it >= 0; it = nx) {   // next item prefetched
                        nx = next_item(&S.head2, ng * SNW * nw, lane);
                        const int wd = it % nw, lw = it / nw, l = lw / SNW, w = lw - l * SNW;
                        if (!S.need[l][w] || !S.wm[(l * SNW + w) * nw + wd]) continue;
                        soft_grad_item<false>(S, S.rec + l * n, S.wm + (l * SNW + w) * nw, nw, l, w, lane, tc, kexp,
                                              c2, wd, wd + 1);
                    }
#else
                    for (int it = next_item(&S.head, ng * SNW, lane), nx = 0; it >= 0; it = nx) {   // next item prefetched
                        nx = next_item(&S.head, ng * SNW, lane);
                        const int l = it / SNW, w = it - l * SNW;
                        if (!S.need[l][w]) continue;
                        soft_grad_item<true>(S, S.rec + l * n, S.wm + (l * SNW + w) * nw, nw, l, w, lane, tc, kexp, c2);
                    }
#endif
                }
                __syncthreads();
            }
            if (touched) {
                flush_slots(S, t, im, ch.s, n, sb.ent);
                __syncthreads();
            }
        } else {
            for (int k = ch.k0; k < ch.k1; ++k) {
                load_need(t, im, k, tile, warp, lane, want, &S.need[0][warp]);
                if (threadIdx.x == 0) S.taus[0] = t.sched_tau[im.sched_off + k];
                S.pnz[0][myp] = 1.f;
                S.nz[0][myp] = 0;
                __syncthreads();
                uint32_t anyn = 0u;
#pragma unroll
                for (int w = 0; w < SNW; ++w) anyn |= S.need[0][w];
                int base = 0, fpos = 0;
                if (t.spz) {   // K8 left the products: one pass, batch by batch
                    const float *pzc = t.spz + ((size_t)(im.cov_off + k) * t.T + tile) * NPX;
                    while (anyn) {
                        const int nb = sb.fb ? soft_fallback_fill(t, sb.rseg, S.taus[0], tc, SREC_B9, fpos, S.sid, S.wsum)
                                             : (base < sb.n ? min(SREC_B9, sb.n - base) : 0);
                        if (nb == 0) break;
                        const int nw = (nb + 31) >> 5;
                        for (int i = threadIdx.x; i < SNW * nw; i += NT) S.wm[i] = 0u;
                        if (threadIdx.x == 0) { S.head2 = 0; S.nitems = 0; }
                        __syncthreads();
                        soft_stage_group<false>(t, sb, nb, base, S.taus, 1, tc, S.need, S.sid, S.rec, S.wm, dummy, t.rcut);
                        __syncthreads();
                        if (S.need[0][warp]) {   // this warp lists its footprint's non-empty batches
                            const unsigned cnt = lane < nw ? __popc(S.wm[warp * nw + lane]) : 0u;
                            const int nbt = (int)((__reduce_add_sync(0xffffffffu, cnt) + 31u) >> 5);
                            int b0 = 0;
                            if (lane == 0 && nbt) b0 = atomicAdd(&S.nitems, nbt);
                            b0 = __shfl_sync(0xffffffffu, b0, 0);
                            if (lane < nbt) S.items[b0 + lane] = (unsigned short)((warp << 4) | lane);
                        }
                        __syncthreads();
                        const int nit = S.nitems;
                        for (int it = next_item(&S.head2, nit, lane), nx = 0; it >= 0; it = nx) {   // next item prefetched
                            nx = next_item(&S.head2, nit, lane);
                            const int v = S.items[it], w = v >> 4;
                            soft_grad_faces(S, S.rec, S.wm + w * nw, nw, v & 15, 0, w, lane, tc, kexp, c2, pzc);
                        }
                        __syncthreads();
                        flush_slots(S, t, im, ch.s, nb, sb.fb ? S.sid : sb.ent + base);
                        base += nb;
                        __syncthreads();
                    }
                    anyn = 0u;
                }
                while (anyn) {   // pass 1 over all batches
                    const int nb = sb.fb ? soft_fallback_fill(t, sb.rseg, S.taus[0], tc, SREC_B9, fpos, S.sid, S.wsum)
                                         : (base < sb.n ? min(SREC_B9, sb.n - base) : 0);
                    if (nb == 0) break;
                    const int nw = (nb + 31) >> 5;
                    for (int i = threadIdx.x; i < SNW * nw; i += NT) S.wm[i] = 0u;
                    if (threadIdx.x == 0) S.head = 0;
                    __syncthreads();
                    soft_stage_group<false>(t, sb, nb, base, S.taus, 1, tc, S.need, S.sid, S.rec, S.wm, dummy, t.rcut);
                    __syncthreads();
                    for (int it = next_item(&S.head, SNW, lane), nx = 0; it >= 0; it = nx) {   // next item prefetched
                        nx = next_item(&S.head, SNW, lane);
                        if ((S.need[0][it] >> lane) & 1u) {
                            int p;
                            float ul, vl, P = 1.f, Pnz = 1.f;
                            int nz = 0;
                            footprint_pixel(it, lane, tc, p, ul, vl);
                            soft_product<false>(S.rec, S.wm + it * nw, nw, ul, vl, kexp, P, Pnz, nz, dummy);
                            S.pnz[0][p] *= Pnz;
                            S.nz[0][p] = (unsigned short)min((int)S.nz[0][p] + nz, 2);
                        }
                    }
                    base += nb;
                    __syncthreads();
                }
                base = 0;
                fpos = 0;
                while (anyn) {   // pass 2: re-stage each batch
                    const int nb = sb.fb ? soft_fallback_fill(t, sb.rseg, S.taus[0], tc, SREC_B9, fpos, S.sid, S.wsum)
                                         : (base < sb.n ? min(SREC_B9, sb.n - base) : 0);
                    if (nb == 0) break;
                    const int nw = (nb + 31) >> 5;
                    for (int i = threadIdx.x; i < SNW * nw; i += NT) S.wm[i] = 0u;
                    if (threadIdx.x == 0) S.head = 0;
                    __syncthreads();
                    soft_stage_group<false>(t, sb, nb, base, S.taus, 1, tc, S.need, S.sid, S.rec, S.wm, dummy, t.rcut);
                    __syncthreads();
                    for (int it = next_item(&S.head, SNW, lane), nx = 0; it >= 0; it = nx) {   // next item prefetched
                        nx = next_item(&S.head, SNW, lane);
                        if (!S.need[0][it]) continue;
                        soft_grad_item<false>(S, S.rec, S.wm + it * nw, nw, 0, it, lane, tc, kexp, c2);
                    }
                    __syncthreads();
                    flush_slots(S, t, im, ch.s, nb, sb.fb ? S.sid : sb.ent + base);
                    base += nb;
                    __syncthreads();
                }
                __syncthreads();
            }
        }
    }
}

}  // namespace

cudaError_t launch_soft_fwd(const Tables &t, float *out, unsigned long long *census, cudaStream_t st)
{
    if (t.B == 0 || t.T == 0) return cudaSuccess;
    const size_t n = (size_t)t.B * t.H * t.W;
    cudaError_t e;
    if (t.F > 0) {
        const int smem = (int)sizeof(SoftFwdSmem);
        if (census) {
            e = cudaFuncSetAttribute(k8_soft_fwd<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            if (e != cudaSuccess) return e;
            k8_soft_fwd<true><<<dim3(t.T, t.B, t.ssplits), NT, smem, st>>>(t, census);
        } else {
            e = cudaFuncSetAttribute(k8_soft_fwd<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            if (e != cudaSuccess) return e;
            k8_soft_fwd<false><<<dim3(t.T, t.B, t.ssplits), NT, smem, st>>>(t, nullptr);
        }
    } else {
        e = cudaMemsetAsync(t.spart, 0, sizeof(float) * n * t.ssplits, st);
        if (e != cudaSuccess) return e;
    }
    const unsigned blocks = (unsigned)std::min<size_t>((n + 255) / 256, 148 * 16);
    k8_soft_reduce<<<blocks, 256, 0, st>>>(t.spart, reinterpret_cast<float4 *>(out), n, t.ssplits);
    return cudaGetLastError();
}

cudaError_t launch_soft_bwd(const Tables &t, const float *grad, cudaStream_t st)
{
    if (t.B == 0 || t.T == 0 || t.F == 0) return cudaSuccess;
    cudaError_t e;
    if (t.spz) {   // bins with K8's cached products first (K9C), then K9 for the rest
        const int smc = (int)sizeof(SoftBwdCSmem);
        e = cudaFuncSetAttribute(k9c_soft_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, smc);
        if (e != cudaSuccess) return e;
        k9c_soft_bwd<<<dim3(t.T, t.B, t.ssplits), NT, smc, st>>>(t, grad);
    }
    const int smem = (int)sizeof(SoftBwdSmem);
    e = cudaFuncSetAttribute(k9_soft_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    k9_soft_bwd<<<dim3(t.T, t.B, t.ssplits), NT, smem, st>>>(t, grad);
    return cudaGetLastError();
}

}  // namespace br

