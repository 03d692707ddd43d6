// k_raster.cu -- K4 fused raster-forward and K6 fused raster-backward.
//
// One CTA = one 16x16 pixel tile of one image; 8 warps, each owning an 8x4 footprint, one pixel per
// thread.  For every chunk of sub-frames the CTA reads the tile's bin (faces sorted by index).
//   stage   every bin face loads its (face, segment) coefficient record ONCE and evaluates it at
//           each sub-frame tau of the chunk (Eq.8 numerators and denominator, Horner in tau: the
//           paper's "compute once, evaluate per sample"), re-centred at the tile centre and
//           sign-normalised by det F(tau), into a 64 B shared-memory record per (tau, face); it
//           also marks, in a per-(tau, warp) bitmask over the bin slots, the warp footprints its
//           per-tau box and edge functions can reach (integer atomicOr).
//   vis     each warp walks the set bits of its mask (faces in index order) and every lane
//           evaluates the three numerators at its pixel centre (2 FMA each), tests coverage by sign
//           (all w_i >= 0), and keeps the nearest face (z-buffer in registers, strict <, lower
//           index wins exact ties, Q7).  No barrier between the sub-frames of a group.
//   shade   fwd: w_i = N_i / |D|, I = sum w_i c_i (Eq.9), accumulated in registers over all
//           sub-frames; the sub-frames never reach HBM.  Output (1/N) sum, written once.
//           bwd: see the comment above k6_raster_bwd.
// Bins that overflowed are regenerated exactly by scanning all faces in index order (slow path); bins
// longer than the shared-memory record capacity are processed per sub-frame in several batches.
// The hard bins are not sorted: the z-buffer compares (depth, face index), which is independent of
// the order the faces are visited in.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include <cuda_pipeline.h>

#include "internal.cuh"
#include "raster_common.cuh"
#include "../../include/blurrast.h"

namespace br {

#ifndef BR_K4_SACC
#define BR_K4_SACC 1       // K4 keeps the pixel sums in shared memory (frees 4 registers in the hot loop)
#endif
#ifndef BR_HALF
#define BR_HALF 0
#endif
#ifndef BR_K4L_PREF
#define BR_K4L_PREF 0   // 1: the next chunk's bin entries are copied to shared memory (cp.async) during the tests
#endif
#ifndef BR_VIS_STREAM
#define BR_VIS_STREAM 1   // 1: the visibility cache is written / read with evict-first (streaming) accesses
#endif
#ifndef BR_K4L_ONELOAD
#define BR_K4L_ONELOAD 0   // 1: each staged pair requests its whole record at once
#endif
#ifndef BR_K4L_LAZY
#define BR_K4L_LAZY 0   // 1: faces turned away are staged by a warp only where its footprint's back list is tested
#endif
#ifndef BR_K4L_GRP
#define BR_K4L_GRP BR_SREC_F   // (face, sub-frame) pairs per k4l group at most (one sub-frame at least)
#endif
#ifndef BR_STAGE_EARLY
#define BR_STAGE_EARLY 0   // 1: stage_tau writes the record before the footprint masks
#endif
#ifndef BR_K4L_MICRO
#define BR_K4L_MICRO 1   // 1: one-instruction warp max of the winners' depths, __frcp_rn for 1/|D|
#endif
#ifndef BR_K4L_MASKBF
#define BR_K4L_MASKBF 1   // 1: the staging's footprint mask without data-dependent loops (all 8 footprints, box bits)
#endif
// Culling footprints: BR_HALF = 1 -> 4x4 pixel blocks (16 per tile, two per warp: the left and right
// halves of its 8x4 pixels iterate their own face masks), 0 -> the warps' 8x4 blocks.
constexpr int FPW_SH = BR_HALF ? 2 : 3, FPW = 1 << FPW_SH;   // footprint width (pixels); height 4
constexpr int NFP = (TW / FPW) * (TH / 4);    // footprints (mask sets) per sub-frame
__device__ __forceinline__ int fp_of(int warp, int lane) { return BR_HALF ? warp * 2 + ((lane >> 2) & 1) : warp; }
// tuning knobs (overridable with -D for A/B builds; defaults measured on C4, profiles/)
#ifndef BR_SREC_F
#define BR_SREC_F 448
#endif
#ifndef BR_SREC_B
#define BR_SREC_B 384   // (256 -> 384: C5 step 378.8 -> 375.1 ms, C4 K6 2.91 -> 2.88 ms)
#endif
#ifndef BR_GMAX_F
#define BR_GMAX_F 16
#endif
#ifndef BR_GMAX_B
#define BR_GMAX_B 4
#endif
#ifndef BR_K4_MINB
#define BR_K4_MINB 5
#endif
#ifndef BR_K6_MINB
#define BR_K6_MINB 4
#endif
constexpr int SREC_F = BR_SREC_F;   // fwd: staged (tau, face) records per CTA (64 B each)
constexpr int SREC_B = BR_SREC_B;   // bwd: staged records per CTA; also the gather's slot limit
constexpr int GMAX_F = BR_GMAX_F;   // max sub-frames staged together
constexpr int GMAX_B = BR_GMAX_B;
static_assert(VIS_MAXN <= SREC_B && VIS_MAXN <= SREC_F, "cached bins must fit both record stages");


// max over the pixel centres of a local rect [x0..x1] x [y0..y1] of the edge function, >= -tol ?
// (tol_i: per-record rounding allowance, see stage_tau)
__device__ __forceinline__ bool rect_reaches_t(const float A[3], const float B[3], const float G[3], const float tol[3],
                                               int x0, int x1, int y0, int y1, const TileCtx &tc)
{
    const float ulmin = (float)(x0 - TW / 2) * tc.sx, ulmax = (float)(x1 - TW / 2) * tc.sx;
    const float vlmin = (float)(TH / 2 - y1) * tc.sy, vlmax = (float)(TH / 2 - y0) * tc.sy;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const float m = G[i] + A[i] * (A[i] > 0.f ? ulmax : ulmin) + B[i] * (B[i] > 0.f ? vlmax : vlmin);
        if (m < -tol[i]) return false;
    }
    return true;
}

__device__ __forceinline__ bool rect_reaches(const float A[3], const float B[3], const float G[3], int x0, int x1,
                                             int y0, int y1, const TileCtx &tc)
{
    const float ulmin = (float)(x0 - TW / 2) * tc.sx, ulmax = (float)(x1 - TW / 2) * tc.sx;
    const float vlmin = (float)(TH / 2 - y1) * tc.sy, vlmax = (float)(TH / 2 - y0) * tc.sy;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const float m = G[i] + (A[i] > 0.f ? A[i] * ulmax : A[i] * ulmin) + (B[i] > 0.f ? B[i] * vlmax : B[i] * vlmin);
        const float tol = 1e-6f * (fabsf(A[i]) * fmaxf(-ulmin, ulmax) + fabsf(B[i]) * fmaxf(-vlmin, vlmax) +
                                   fabsf(G[i])) + 1e-30f;
        if (m < -tol) return false;
    }
    return true;
}

// Evaluate a record at tau for this tile -> TauRec + the mask of warp footprints it can reach
// (bit w = culling footprint w, see FPW; 0 = the face cannot cover any pixel of the tile at tau).
// D = det F(tau) (|D| > EPS_D) and the face's pixel box in the tile come from the caller's rejects.
template <bool GRID, bool BOXONLY = false, bool R48 = false>
__device__ __forceinline__ uint32_t stage_tau(const FaceRec &fr, float tau, float D, int x0, int x1, int y0, int y1,
                                              const TileCtx &tc, TauRec &out, float4 *d48 = nullptr,
                                              float2 *x48 = nullptr)
{
    // R48: the record goes to d48[0..2] (TauRec's first 48 bytes, in its order) and (invD, face) to *x48; out unused
    const float4 q6 = fr.q[6];
    const float sg = D < 0.f ? -1.f : 1.f;
    const float invD = BR_K4L_MICRO ? __frcp_rn(fabsf(D)) : 1.0f / fabsf(D);   // the same correctly rounded value
    float A[3], B[3], G[3];
    const float *ef = reinterpret_cast<const float *>(fr.q);
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        float al, be, gp;
        rec_edge_at(fr.q[2 * i], fr.q[2 * i + 1], tau, tc.uc, tc.vc, al, be, gp);
        A[i] = al * sg;
        B[i] = be * sg;
        G[i] = gp * sg;
    }
#if BR_STAGE_EARLY
    {   // the record first (its slot is this pair's own; unused when no footprint is reached): the record's
        // registers die before the footprint masks need theirs (fewer spills under the 48-register cap)
        const float4 z0 = fr.q[9], z1 = fr.q[10];
        const float za = __fmaf_rn(tau, z1.x - z0.x, z0.x);
        const float zb = __fmaf_rn(tau, z1.y - z0.y, z0.y);
        const float zc = __fmaf_rn(tau, z1.z - z0.z, z0.z);
        out.a[0] = A[0]; out.a[1] = A[1]; out.a[2] = A[2];
        out.b[0] = B[0]; out.b[1] = B[1]; out.b[2] = B[2];
        out.g[0] = G[0]; out.g[1] = G[1]; out.g[2] = G[2];
        const float dzb = zb - za, dzc = zc - za;
        out.az = __fmaf_rn(A[1], dzb, A[2] * dzc) * invD;
        out.bz = __fmaf_rn(B[1], dzb, B[2] * dzc) * invD;
        out.cz = __fmaf_rn(__fmaf_rn(G[1], dzb, G[2] * dzc), invD, za);
        out.invD = invD;
        out.fid = __float_as_int(q6.w);
    }
#endif
    // culling footprints (FPW x 4) reached by the box and the three edge half-planes; the
    // rounding allowance is bounded once over the whole tile (|ul|, |vl| <= 8 pixels)
    float tol[3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
        tol[i] = 1e-6f * (fabsf(A[i]) * (8.f * tc.sx) + fabsf(B[i]) * (8.f * tc.sy) + fabsf(G[i])) + 1e-30f;
    // the max of e_i over a footprint rect (clipped to the box) sits at the corner along (A_i, B_i): a
    // column term A_i u per footprint column of the box, a row term G_i + B_i v + tol_i per row, and the
    // footprint is reached iff every edge has column + row term >= 0
    uint32_t fm = 0u;
    if (BOXONLY) {   // the footprints the box reaches (a superset: more footprint tests, a cheaper stage)
        for (int wy = y0 >> 2; wy <= (y1 >> 2); ++wy)
            for (int wx = x0 >> FPW_SH; wx <= (x1 >> FPW_SH); ++wx) fm |= 1u << (wy * (TW / FPW) + wx);
    } else if (!GRID) {   // per footprint (K6's copy: keeps that kernel's register allocation)
        for (int wy = y0 >> 2; wy <= (y1 >> 2); ++wy)
            for (int wx = x0 >> FPW_SH; wx <= (x1 >> FPW_SH); ++wx) {
                const int rx0 = max(x0, wx * FPW), rx1 = min(x1, wx * FPW + FPW - 1);
                const int ry0 = max(y0, wy * 4), ry1 = min(y1, wy * 4 + 3);
                if (rect_reaches_t(A, B, G, tol, rx0, rx1, ry0, ry1, tc)) fm |= 1u << (wy * (TW / FPW) + wx);
            }
    } else if (BR_K4L_MASKBF && !BR_HALF) {
        // branch-free: all 2 x 4 footprints of the tile, each rect clipped to the box (empty rows / columns
        // give a rect outside the box and are masked off by the box bits); the same max-corner test
    const int wx0 = x0 >> 3, wx1 = x1 >> 3, wy0 = y0 >> 2, wy1 = y1 >> 2;
    float cu0[3], cu1[3];
    {
        const float ul00 = (float)(max(x0, 0) - TW / 2) * tc.sx, ul01 = (float)(min(x1, 7) - TW / 2) * tc.sx;
        const float ul10 = (float)(max(x0, 8) - TW / 2) * tc.sx, ul11 = (float)(min(x1, 15) - TW / 2) * tc.sx;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            cu0[i] = A[i] * (A[i] > 0.f ? ul01 : ul00);
            cu1[i] = A[i] * (A[i] > 0.f ? ul11 : ul10);
        }
    }
    const uint32_t colm = (wx0 == 0 ? 1u : 0u) | (wx1 == 1 ? 2u : 0u);
#pragma unroll
    for (int wy = 0; wy < 4; ++wy) {
        const float vlmin = (float)(TH / 2 - min(y1, wy * 4 + 3)) * tc.sy;
        const float vlmax = (float)(TH / 2 - max(y0, wy * 4)) * tc.sy;
        float rv[3];
#pragma unroll
        for (int i = 0; i < 3; ++i) rv[i] = G[i] + B[i] * (B[i] > 0.f ? vlmax : vlmin) + tol[i];
        const bool c0 = rv[0] + cu0[0] >= 0.f && rv[1] + cu0[1] >= 0.f && rv[2] + cu0[2] >= 0.f;
        const bool c1 = rv[0] + cu1[0] >= 0.f && rv[1] + cu1[1] >= 0.f && rv[2] + cu1[2] >= 0.f;
        const uint32_t rowm = (wy >= wy0 && wy <= wy1) ? colm : 0u;
        fm |= (((c0 ? 1u : 0u) | (c1 ? 2u : 0u)) & rowm) << (2 * wy);
    }
    } else {
    const int wx0 = x0 >> FPW_SH, ncol = (x1 >> FPW_SH) - wx0 + 1;
    float cu[TW / FPW][3];
#pragma unroll
    for (int c = 0; c < TW / FPW; ++c) {
        const int wx = min(wx0 + c, TW / FPW - 1);
        const float ulmin = (float)(max(x0, wx * FPW) - TW / 2) * tc.sx;
        const float ulmax = (float)(min(x1, wx * FPW + FPW - 1) - TW / 2) * tc.sx;
#pragma unroll
        for (int i = 0; i < 3; ++i) cu[c][i] = A[i] * (A[i] > 0.f ? ulmax : ulmin);
    }
    for (int wy = y0 >> 2; wy <= (y1 >> 2); ++wy) {
        const float vlmin = (float)(TH / 2 - min(y1, wy * 4 + 3)) * tc.sy;
        const float vlmax = (float)(TH / 2 - max(y0, wy * 4)) * tc.sy;
        float rv[3];
#pragma unroll
        for (int i = 0; i < 3; ++i) rv[i] = G[i] + B[i] * (B[i] > 0.f ? vlmax : vlmin) + tol[i];
#pragma unroll
        for (int c = 0; c < TW / FPW; ++c)
            if (c < ncol && rv[0] + cu[c][0] >= 0.f && rv[1] + cu[c][1] >= 0.f && rv[2] + cu[c][2] >= 0.f)
                fm |= 1u << (wy * (TW / FPW) + wx0 + c);
    }
    }
    if (!fm || BR_STAGE_EARLY) return fm;
    const float4 z0 = fr.q[9], z1 = fr.q[10];
    const float za = __fmaf_rn(tau, z1.x - z0.x, z0.x);
    const float zb = __fmaf_rn(tau, z1.y - z0.y, z0.y);
    const float zc = __fmaf_rn(tau, z1.z - z0.z, z0.z);
    if (!R48) {
        out.a[0] = A[0]; out.a[1] = A[1]; out.a[2] = A[2];
        out.b[0] = B[0]; out.b[1] = B[1]; out.b[2] = B[2];
        out.g[0] = G[0]; out.g[1] = G[1]; out.g[2] = G[2];
    }
    // depth interpolated with the screen-space weights (Q6): z(p) = sum_i w_i(p) z_i, written as
    // z0 + w1 (z1 - z0) + w2 (z2 - z0).  Same plane when sum_i w_i = 1; in fp32 the weights of a
    // sliver face sum to 1 +- 1e-4, and this form keeps that error off the absolute depth.
    const float dzb = zb - za, dzc = zc - za;
    if (R48) {
        const float az = __fmaf_rn(A[1], dzb, A[2] * dzc) * invD;
        const float bz = __fmaf_rn(B[1], dzb, B[2] * dzc) * invD;
        const float cz = __fmaf_rn(__fmaf_rn(G[1], dzb, G[2] * dzc), invD, za);
        d48[0] = make_float4(A[0], A[1], A[2], B[0]);
        d48[1] = make_float4(B[1], B[2], G[0], G[1]);
        d48[2] = make_float4(G[2], az, bz, cz);
        *x48 = make_float2(invD, q6.w);
        return fm;
    }
    out.az = __fmaf_rn(A[1], dzb, A[2] * dzc) * invD;
    out.bz = __fmaf_rn(B[1], dzb, B[2] * dzc) * invD;
    out.cz = __fmaf_rn(__fmaf_rn(G[1], dzb, G[2] * dzc), invD, za);
    out.invD = invD;
    out.fid = __float_as_int(q6.w);
    return fm;
}

// The record of a (face, sub-frame) for this tile without its footprint mask: the same arithmetic as stage_tau
// (bit-identical TauRec), for the lazily staged faces turned away from the camera (BR_K4L_LAZY).
__device__ __forceinline__ void rec_at(const FaceRec &fr, float tau, float D, const TileCtx &tc, TauRec &out)
{
    const float4 q6 = fr.q[6];
    const float sg = D < 0.f ? -1.f : 1.f;
    const float invD = BR_K4L_MICRO ? __frcp_rn(fabsf(D)) : 1.0f / fabsf(D);
    float A[3], B[3], G[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        float al, be, gp;
        rec_edge_at(fr.q[2 * i], fr.q[2 * i + 1], tau, tc.uc, tc.vc, al, be, gp);
        A[i] = al * sg;
        B[i] = be * sg;
        G[i] = gp * sg;
    }
    const float4 z0 = fr.q[9], z1 = fr.q[10];
    const float za = __fmaf_rn(tau, z1.x - z0.x, z0.x);
    const float zb = __fmaf_rn(tau, z1.y - z0.y, z0.y);
    const float zc = __fmaf_rn(tau, z1.z - z0.z, z0.z);
    out.a[0] = A[0]; out.a[1] = A[1]; out.a[2] = A[2];
    out.b[0] = B[0]; out.b[1] = B[1]; out.b[2] = B[2];
    out.g[0] = G[0]; out.g[1] = G[1]; out.g[2] = G[2];
    const float dzb = zb - za, dzc = zc - za;
    out.az = __fmaf_rn(A[1], dzb, A[2] * dzc) * invD;
    out.bz = __fmaf_rn(B[1], dzb, B[2] * dzc) * invD;
    out.cz = __fmaf_rn(__fmaf_rn(G[1], dzb, G[2] * dzc), invD, za);
    out.invD = invD;
    out.fid = __float_as_int(q6.w);
}

// NEXT-2 ablation (the paper's per-frame baseline): instead of evaluating
// the per-segment coefficients, lerp the three keyframe vertices to tau (Eq.5-6) and set the
// triangle up from scratch for this sub-frame (edge functions = rows of adj F(tau), det F(tau)).
// solver 1 ("naive per-frame") keeps the same per-pixel work as the fast path; solver 2 ("naive
// per-pixel") additionally stores the lerped vertices so that every (pixel, face, sub-frame) test
// re-solves w = F(tau)^-1 p (Eq.3) -- the SoftRas-style cost the paper accelerates.
template <int MODE>
__device__ __forceinline__ uint32_t stage_tau_naive(const BinCtx &bc, int f, float tau, const TileCtx &tc, int W,
                                                    int H, TauRec &out, float4 *vout)
{
    const float4 q = __ldg(bc.fcol + 3 * (size_t)f + 2);
    const int vid[3] = {__float_as_int(q.y), __float_as_int(q.z), __float_as_int(q.w)};
    float X[3], Y[3], Z[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const float4 a = __ldg(bc.key0 + vid[i]), b = __ldg(bc.key1 + vid[i]);
        X[i] = __fsub_rn(__fmaf_rn(tau, __fsub_rn(b.x, a.x), a.x), tc.uc);     // tile-centred
        Y[i] = __fsub_rn(__fmaf_rn(tau, __fsub_rn(b.y, a.y), a.y), tc.vc);
        Z[i] = __fmaf_rn(tau, b.z - a.z, a.z);
    }
    const float D = __fsub_rn(__fmul_rn(__fsub_rn(X[1], X[0]), __fsub_rn(Y[2], Y[0])),
                              __fmul_rn(__fsub_rn(Y[1], Y[0]), __fsub_rn(X[2], X[0])));
    if (!(fabsf(D) > EPS_D)) return 0u;
    const float xmn = fminf(fminf(X[0], X[1]), X[2]) + tc.uc - BBOX_PAD, xmx = fmaxf(fmaxf(X[0], X[1]), X[2]) + tc.uc + BBOX_PAD;
    const float ymn = fminf(fminf(Y[0], Y[1]), Y[2]) + tc.vc - BBOX_PAD, ymx = fmaxf(fmaxf(Y[0], Y[1]), Y[2]) + tc.vc + BBOX_PAD;
    int x0, x1, y0, y1;
    if (!tile_pixels(xmn, xmx, ymn, ymx, W, H, tc, x0, x1, y0, y1)) return 0u;
    const float sg = D < 0.f ? -1.f : 1.f;
    const float invD = 1.0f / fabsf(D);
    float A[3], B[3], G[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {   // edge opposite corner i, canonical direction (lower vertex id first)
        const int j = (i + 1) % 3, l = (i + 2) % 3;
        const bool fwd = vid[j] < vid[l];
        const int a = fwd ? j : l, c = fwd ? l : j;
        const float ex = __fsub_rn(X[c], X[a]), ey = __fsub_rn(Y[c], Y[a]);
        const float g = __fsub_rn(__fmul_rn(X[a], ey), __fmul_rn(Y[a], ex));   // N at the tile centre
        const float cs = (fwd ? 1.f : -1.f) * sg;
        A[i] = -ey * cs;
        B[i] = ex * cs;
        G[i] = g * cs;
    }
    uint32_t fm = 0u;
    for (int wy = y0 >> 2; wy <= (y1 >> 2); ++wy)
        for (int wx = x0 >> FPW_SH; wx <= (x1 >> FPW_SH); ++wx) {
            const int rx0 = max(x0, wx * FPW), rx1 = min(x1, wx * FPW + FPW - 1);
            const int ry0 = max(y0, wy * 4), ry1 = min(y1, wy * 4 + 3);
            if (rect_reaches(A, B, G, rx0, rx1, ry0, ry1, tc)) fm |= 1u << (wy * (TW / FPW) + wx);
        }
    if (!fm) return 0u;
    out.a[0] = A[0]; out.a[1] = A[1]; out.a[2] = A[2];
    out.b[0] = B[0]; out.b[1] = B[1]; out.b[2] = B[2];
    out.g[0] = G[0]; out.g[1] = G[1]; out.g[2] = G[2];
    const float dzb = Z[1] - Z[0], dzc = Z[2] - Z[0];
    out.az = __fmaf_rn(A[1], dzb, A[2] * dzc) * invD;
    out.bz = __fmaf_rn(B[1], dzb, B[2] * dzc) * invD;
    out.cz = __fmaf_rn(__fmaf_rn(G[1], dzb, G[2] * dzc), invD, Z[0]);
    out.invD = invD;
    out.fid = f;
    if (MODE == 2) {
        vout[0] = make_float4(X[0], Y[0], Z[0], X[1]);
        vout[1] = make_float4(Y[1], Z[1], X[2], Y[2]);
        vout[2] = make_float4(Z[2], 0.f, 0.f, 0.f);
    }
    return fm;
}

// Stage faces [base, base+nb) of the bin (or sid[] in fallback mode) at the ng sub-frames
// taus[0..ng): records rec[l*nb + j], masks wm[(l*NFP + w)*nw + j/32].  Masks must be clear.
// Work is spread over (face, sub-frame) pairs, face-major, so the lanes that share a face load its
// record with broadcast loads.
template <bool CENSUS, int MODE, bool GRID = false>
__device__ __forceinline__ void stage_group(const BinCtx &bc, int nb, int base, const float *taus, int ng,
                                            const TileCtx &tc, int W, int H, int F, const int *sid, TauRec *rec,
                                            float4 *vtx, uint32_t *wm, unsigned long long &nstage)
{
    const int nw = (nb + 31) >> 5;
    const int npair = nb * ng;
    const float inv_ng = 1.0f / (float)ng;
    for (int p = threadIdx.x; p < npair; p += NT) {
        const int j = div_small(p, inv_ng), l = p - j * ng;
        const int f = bc.fb ? sid[j] : __ldg(bc.ent + base + j);
        if ((unsigned)f >= (unsigned)F) {     // never expected: bins hold valid face ids
#ifdef BR_DEBUG
            printf("bad face id %d (F=%d) fb=%d n=%d base=%d j=%d nb=%d tile=%d img=%d\n", f, F, (int)bc.fb, bc.n,
                   base, j, nb, blockIdx.x, blockIdx.y);
#endif
            atomicOr(bc.status, BLUR_ST_EINTERNAL);
            continue;
        }
        const float4 *r = bc.rseg + (size_t)f * REC_F4;
        const float4 q6 = __ldg(r + 6);
        if (__float_as_int(q6.w) < 0) continue;               // skipped face (Q8, behind, bad index)
        const float tau = taus[l];
        // cheap rejects before the full record is loaded: degenerate at tau (Q8), box off the tile
        const float D = __fmaf_rn(tau, __fmaf_rn(tau, q6.x, q6.y), q6.z);   // a1 t^2 + a2 t + a3
        if (!(fabsf(D) > EPS_D)) continue;
        const float4 b0 = __ldg(r + 7), b1 = __ldg(r + 8);
        int x0, x1, y0, y1;
        if (!tile_pixels(box_lerp(tau, b0.x, b1.x), box_lerp(tau, b0.y, b1.y), box_lerp(tau, b0.z, b1.z),
                         box_lerp(tau, b0.w, b1.w), W, H, tc, x0, x1, y0, y1))
            continue;
        uint32_t fm;
        if (MODE == 0) {
            FaceRec fr;
            load_rec(r, fr);
            fm = stage_tau<GRID>(fr, tau, D, x0, x1, y0, y1, tc, rec[l * nb + j]);
        } else {
            fm = stage_tau_naive<MODE>(bc, f, tau, tc, W, H, rec[l * nb + j], vtx + 3 * (l * nb + j));
        }
        if (CENSUS) nstage += fm != 0u;
        const uint32_t bit = 1u << (j & 31);
        for (uint32_t m = fm; m; m &= m - 1) atomicOr(wm + (l * NFP + (__ffs(m) - 1)) * nw + (j >> 5), bit);
    }
}

// Visibility of one pixel over the faces of its warp's mask (any visiting order): z-buffer on
// (depth, face index).  vis_mask_fast keeps strict < on depth only and reports whether an exact depth
// tie occurred (the caller then re-runs vis_mask, which compares face indices) -- ties need exactly
// equal float depths of two faces at a pixel centre, so the common loop stays short.
template <bool CENSUS, int MODE>
__device__ __forceinline__ bool vis_mask_fast(const TauRec *rec, const uint32_t *wm, int nw, float ul, float vl,
                                              float &zbest, int &ebest, unsigned long long &ncov,
                                              unsigned long long &ntest, bool count)
{
    float tief = 0.f;
    // words walked by pointer with a countdown (a `wd < nw` bound or an end pointer was re-derived
    // from the bin length at every word under register pressure)
    const uint32_t *wp = wm;
    const float4 *rw = reinterpret_cast<const float4 *>(rec);
    for (int wbase = 0, left = nw; left > 0; --left, ++wp, rw += 4 * 32, wbase += 32) {
        uint32_t m = *wp;
        while (m) {
            int k;
            asm("bfind.u32 %0, %1;" : "=r"(k) : "r"(m));   // highest set bit (any order is fine)
            m ^= 1u << k;
            const float4 *rp = rw + 4 * k;
            const float4 q0 = rp[0], q1 = rp[1], q2 = rp[2];
            const float e0 = edge_eval(q0.x, q0.w, q1.z, ul, vl);
            const float e1 = edge_eval(q0.y, q1.x, q1.w, ul, vl);
            const float e2 = edge_eval(q0.z, q1.y, q2.x, ul, vl);
            const float z = __fmaf_rn(q2.y, ul, __fmaf_rn(q2.z, vl, q2.w));
            const float emin = fminf(fminf(e0, e1), e2);
            if (CENSUS && count) { ncov += emin >= 0.f; ntest += 1; }
            // covered with z == zbest: an exact depth tie (kept in a float: one FSEL per test)
            tief = (emin >= 0.f && z == zbest) ? 1.f : tief;
            if (emin >= 0.f && z < zbest) { zbest = z; ebest = wbase + k; }
        }
    }
    return tief != 0.f;
}

template <bool CENSUS, int MODE>
__device__ __forceinline__ void vis_mask(const TauRec *rec, const float4 *vtx, const uint32_t *wm, int nw,
                                         int ebase, float ul, float vl, float &zbest, int &ebest, int &fbest,
                                         unsigned long long &ncov, unsigned long long &ntest, bool count)
{
    for (int wd = 0; wd < nw; ++wd) {
        uint32_t m = wm[wd];
        const TauRec *rw = rec + (wd << 5);
        while (m) {
            const int k = 31 - __clz(m);
            m ^= 1u << k;
            const int j = (wd << 5) + k;
            bool cov;
            float z;
            if (MODE != 2) {
                const float4 *rp = reinterpret_cast<const float4 *>(rw + k);
                const float4 q0 = rp[0], q1 = rp[1], q2 = rp[2];
                const float e0 = edge_eval(q0.x, q0.w, q1.z, ul, vl);
                const float e1 = edge_eval(q0.y, q1.x, q1.w, ul, vl);
                const float e2 = edge_eval(q0.z, q1.y, q2.x, ul, vl);
                z = __fmaf_rn(q2.y, ul, __fmaf_rn(q2.z, vl, q2.w));
                cov = fminf(fminf(e0, e1), e2) >= 0.f;
            } else {
                // per-pixel textbook solve w = F(tau)^-1 p (Eq.3): sub-triangle areas over det F
                const float4 a = vtx[3 * j], b = vtx[3 * j + 1], c = vtx[3 * j + 2];
                const float dx0 = a.x - ul, dy0 = a.y - vl, dx1 = a.w - ul, dy1 = b.x - vl, dx2 = b.z - ul,
                            dy2 = b.w - vl;
                const float n0 = __fsub_rn(__fmul_rn(dx1, dy2), __fmul_rn(dx2, dy1));
                const float n1 = __fsub_rn(__fmul_rn(dx2, dy0), __fmul_rn(dx0, dy2));
                const float n2 = __fsub_rn(__fmul_rn(dx0, dy1), __fmul_rn(dx1, dy0));
                const float det = n0 + n1 + n2;
                const float id = 1.0f / det;
                const float w0 = n0 * id, w1 = n1 * id, w2 = n2 * id;
                z = w0 * a.z + w1 * b.y + w2 * c.x;
                cov = fminf(fminf(w0, w1), w2) >= 0.f && det != 0.f;
            }
            if (CENSUS && count) { ncov += cov; ntest += 1; }
            // z-buffer on (depth, face index): strict < in depth, the lower face index on exact ties
            // (Q7) -- order-independent, so the bins need not be sorted
            if (cov && z <= zbest) {
                const int fj = rw[k].fid;
                if (z < zbest || fj < fbest) { zbest = z; ebest = ebase + j; fbest = fj; }
            }
        }
    }
}


__device__ __forceinline__ void clear_words(uint32_t *w, int n)
{
    for (int i = threadIdx.x; i < n; i += NT) w[i] = 0u;
}

template <int MODE>
struct FwdSmem {
    TauRec rec[SREC_F];
    float4 vtx[MODE == 2 ? 3 * SREC_F : 1];   // solver 2: lerped vertices per staged record
    uint32_t wm[NFP * (SREC_F / 32 + GMAX_F)];
    int sid[SREC_F];
    float taus[GMAX_F];
    int wsum[NWARP];
#if BR_K4_SACC
    float4 acc[TW * TH];   // per-pixel (r, g, b, a) sums over the sub-frames (thread-private slot)
#endif
    float2 uv[NT];         // the thread's pixel (ul, vl): reloaded at each visibility pass instead of being
                           // re-derived from the thread index under register pressure
};

template <bool CENSUS, int MODE>
__global__ void __launch_bounds__(NT, BR_K4_MINB) k4_raster_fwd(Tables t, float *__restrict__ out, int *__restrict__ ids,
                                                       int ids_k, unsigned long long *census)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    FwdSmem<MODE> &S = *reinterpret_cast<FwdSmem<MODE> *>(smem_raw);
    const int b = blockIdx.y, tile = blockIdx.x;
    const ImgInfo &im = t.imgs[b];
    const int N = im.N, c_begin = im.chunk_begin, c_end = im.chunk_end, sched_off = im.sched_off;
    const long long rec_off = im.rec_off;
    TileCtx tc;
    tile_ctx(t, tile, tc);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int lx = (warp & 1) * 8 + (lane & 7), ly = (warp >> 1) * 4 + (lane >> 3);
    const int px = tc.px0 + lx, py = tc.py0 + ly;
    const bool inimg = px < t.W && py < t.H;
    const float ul = (float)(lx - TW / 2) * tc.sx;
    const float vl = (float)(TH / 2 - ly) * tc.sy;
#define PIX (((size_t)b * t.H + py) * t.W + px)   // (recomputed where used: keeps registers free)
    const int myp = ly * TW + lx;
    S.uv[threadIdx.x] = make_float2(ul, vl);
#if BR_K4_SACC
    S.acc[myp] = make_float4(0.f, 0.f, 0.f, 0.f);
#define K4_ACC(pr, pg, pb) do { float4 a_ = S.acc[myp]; a_.x += (pr); a_.y += (pg); a_.z += (pb); a_.w += 1.f; S.acc[myp] = a_; } while (0)
#else
    float ar = 0.f, ag = 0.f, ab = 0.f, aa = 0.f;
#define K4_ACC(pr, pg, pb) do { ar += (pr); ag += (pg); ab += (pb); aa += 1.f; } while (0)
#endif
    unsigned long long ncov = 0, ntest = 0, nshade = 0, nstage = 0;

    for (int c = c_begin + (int)blockIdx.z; c < c_end; c += t.splits) {
        const Chunk ch = t.chunks[c];
        const size_t bi = (size_t)c * t.T + tile;
        const long long o = t.off[bi];
        const int n = (int)(t.off[bi + 1] - o);
        if (n == 0) {
            if (ids && inimg && ids_k >= ch.k0 && ids_k < ch.k1) ids[PIX] = -1;
            if (t.covbits) {
                const unsigned m = __ballot_sync(0xffffffffu, !inimg);
                if (lane == 0)
                    for (int k = ch.k0; k < ch.k1; ++k) t.covbits[cov_word(t, im, k, tile) + warp] = m;
            }
            continue;
        }
        BinCtx bc;
        bc.status = t.status;
        bc.rseg = t.rec + (size_t)(rec_off + (long long)ch.s * t.F) * REC_F4;
        bc.key0 = t.key + im.key_off + (size_t)ch.s * t.V;
        bc.key1 = bc.key0 + t.V;
        bc.fcol = t.fcol;
        bc.ent = t.entries + o;
        bc.n = n;
        bc.fb = o + n > t.cap;
        if (!bc.fb && n <= SREC_F) {
            // grouped path: the whole bin staged for up to Gs sub-frames at once
            const int Gs = min(GMAX_F, SREC_F / n), nw = (n + 31) >> 5;
            uint16_t *vis_out = (MODE == 0 && n <= VIS_MAXN) ? t.vis : nullptr;
            for (int kg = ch.k0; kg < ch.k1; kg += Gs) {
                const int ng = min(Gs, ch.k1 - kg);
                clear_words(S.wm, ng * NFP * nw);
                if (threadIdx.x < ng) S.taus[threadIdx.x] = t.sched_tau[sched_off + kg + threadIdx.x];
                __syncthreads();
                stage_group<CENSUS, MODE, true>(bc, n, 0, S.taus, ng, tc, t.W, t.H, t.F, S.sid, S.rec, S.vtx, S.wm, nstage);
                __syncthreads();
                // visibility-buffer row of this pixel at sub-frame kg, advanced by one sub-frame per l
                uint16_t *vrow = vis_out ? vis_out + ((size_t)(im.cov_off + kg) * t.T + tile) * (TW * TH) + myp : nullptr;
                const int l_ids = (ids && inimg) ? ids_k - kg : -1;
                for (int l = 0; l < ng; ++l) {
                    float zbest = __int_as_float(0x7f800000);
                    int ebest = -1, fbest = 0x7fffffff;
                    const TauRec *rl = S.rec + l * n;
                    const uint32_t *wml = S.wm + (l * NFP + fp_of(warp, lane)) * nw;
                    bool tie = true;
                    if (MODE != 2) {
                        const float2 uv = S.uv[threadIdx.x];
                        tie = vis_mask_fast<CENSUS, MODE>(rl, wml, nw, uv.x, uv.y, zbest, ebest, ncov, ntest, inimg);
                    }
                    if (__any_sync(0xffffffffu, tie)) {   // exact depth tie somewhere in the warp: face indices decide
                        unsigned long long d0 = 0, d1 = 0;
                        zbest = __int_as_float(0x7f800000);
                        ebest = -1;
                        if (MODE != 2) vis_mask<false, MODE>(rl, S.vtx + 3 * l * n, wml, nw, 0, ul, vl, zbest, ebest, fbest, d0, d1, false);
                        else vis_mask<CENSUS, MODE>(rl, S.vtx + 3 * l * n, wml, nw, 0, ul, vl, zbest, ebest, fbest, ncov, ntest, inimg);
                    }
                    int fid = -1;
                    if (ebest >= 0) {
                        float pr, pg, pb;
                        shade(rl[ebest], t.fcol, ul, vl, pr, pg, pb);      // Eq.9
                        K4_ACC(pr, pg, pb);
                        fid = rl[ebest].fid;
                        if (CENSUS) nshade++;
                    }
                    if (l == l_ids) ids[PIX] = fid;
                    if (vrow) {   // visibility buffer for K6 (bins it takes the grouped path for)
                        *vrow = ebest >= 0 ? (uint16_t)ebest : (uint16_t)0xFFFF;
                        vrow += (size_t)t.T * (TW * TH);
                    }
                    if (t.covbits) {   // soft path: which pixels of the warp are covered at this sub-frame
                        const unsigned m = __ballot_sync(0xffffffffu, ebest >= 0 || !inimg);
                        if (lane == 0) t.covbits[cov_word(t, im, kg + l, tile) + warp] = m;
                    }
                }
                __syncthreads();
            }
        } else {
            // per sub-frame, several batches (long bins) or the exact fallback scan (overflow)
            for (int k = ch.k0; k < ch.k1; ++k) {
                const float tau = t.sched_tau[sched_off + k];
                float zbest = __int_as_float(0x7f800000);
                int ebest = -1, bfid = -1, fbest = 0x7fffffff;
                bool has = false;
                float pr = 0.f, pg = 0.f, pb = 0.f;
                int base = 0, fpos = 0;
                if (threadIdx.x == 0) S.taus[0] = tau;
                while (true) {
                    const int nb = next_batch(bc, t.F, tau, tc, t.W, t.H, SREC_F, base, fpos, S.sid, S.wsum);
                    if (nb == 0) break;
                    const int nw = (nb + 31) >> 5;
                    clear_words(S.wm, NFP * nw);
                    __syncthreads();
                    stage_group<CENSUS, MODE, true>(bc, nb, base, S.taus, 1, tc, t.W, t.H, t.F, S.sid, S.rec, S.vtx, S.wm, nstage);
                    __syncthreads();
                    vis_mask<CENSUS, MODE>(S.rec, S.vtx, S.wm + fp_of(warp, lane) * nw, nw, base, ul, vl, zbest, ebest, fbest, ncov,
                                           ntest, inimg);
                    if (ebest >= base) {   // winner changed in this batch: shade now (Eq.9)
                        shade(S.rec[ebest - base], t.fcol, ul, vl, pr, pg, pb);
                        has = true;
                        bfid = S.rec[ebest - base].fid;
                        fbest = bfid;      // ties against later batches compare face indices
                    }
                    base += nb;
                    __syncthreads();
                }
                if (has) { K4_ACC(pr, pg, pb); if (CENSUS) nshade++; }
                if (ids && inimg && k == ids_k) ids[PIX] = has ? bfid : -1;
                if (t.covbits) {
                    const unsigned m = __ballot_sync(0xffffffffu, has || !inimg);
                    if (lane == 0) t.covbits[cov_word(t, im, k, tile) + warp] = m;
                }
            }
        }
    }
    if (inimg && out) {   // out == null: coverage-only pass (soft backward without a preceding forward)
        const float inv = 1.0f / (float)N;
#if BR_K4_SACC
        const float4 a = S.acc[myp];
        const float4 v = make_float4(a.x * inv, a.y * inv, a.z * inv, a.w * inv);
#else
        const float4 v = make_float4(ar * inv, ag * inv, ab * inv, aa * inv);
#endif
        if (t.splits == 1) reinterpret_cast<float4 *>(out)[PIX] = v;
        else t.part[(size_t)blockIdx.z * ((size_t)t.B * t.H * t.W) + PIX] = v;
    }
#undef PIX
    if (CENSUS) {
        atomicAdd(census + 0, ncov);
        atomicAdd(census + 1, inimg ? nshade : 0ull);
        atomicAdd(census + 2, ntest);
        atomicAdd(census + 3, nstage);
    }
}

// ------------------------------------------------------------------ lean forward (fast solver)
//
// k4l_raster_fwd: K4 for the fast solver without the census (the timed path).  The same stage, tests and
// shading as k4_raster_fwd, but each (sub-frame, warp footprint) gets a compact list of the bin slots
// whose record reaches it (shared atomic counters in the stage) instead of a bitmask over all slots:
// the visibility loop walks exactly the reaching records, with no per-word walk over the mostly empty
// mask words of long bins, and the per-(warp, sub-frame) bookkeeping is kept in registers.  Long and
// overflowed bins take k4_raster_fwd's per-sub-frame batch path unchanged.

#ifndef BR_K4L_UNIT
#define BR_K4L_UNIT 0   // 1: staging units of (face, block of sub-frames), one record load per unit (C4 K4 6.14 -> 8.09 ms)
#endif
#ifndef BR_K4L_PAIR2
#define BR_K4L_PAIR2 0  // 1: two pairs per thread, both pairs' first record words requested together (measured slower)
#endif
#ifndef BR_K4L_TWOPASS
#define BR_K4L_TWOPASS 0   // 1: box tests first, then the full stage over the compacted accepted pairs (C4 6.88 -> 7.51 ms)
#endif
#ifndef BR_K4L_SENT
#define BR_K4L_SENT 0   // 1: the chunk's bin entries staged in shared memory (measured: no change)
#endif
#ifndef BR_K4L_BACKBOX
#define BR_K4L_BACKBOX 0   // 1: faces turned away from the camera get footprints from the box only (C4 K4 6.14 -> 6.38 ms)
#endif
#ifndef BR_K4L_UNROLL
#define BR_K4L_UNROLL 0
#endif
#if BR_K4L_UNROLL
#define BR_UNROLL4 _Pragma("unroll 4")
#else
#define BR_UNROLL4
#endif
#ifndef BR_K4L_TPREF
#define BR_K4L_TPREF 0   // 1: the next chunk's header / bin offsets and the next group's taus are requested one phase
                         // ahead (registers), so that no global load sits between two barriers (measured: C4 K4
                         // 5.86 -> 5.96 ms, 16 B more spill loads; parity-green)
#endif
#ifndef BR_K4L_NWIN
#define BR_K4L_NWIN 0   // 1: the bin sizes of the CTA's next 32 chunks are loaded at once (lane j: chunk j), so that
                        // empty bins cost no L2 round trip each (measured: C4 K4 5.86 -> 5.95 ms, C3 1.25 -> 1.26;
                        // parity-green: the empty-bin round trips are hidden by the other CTAs of the SM)
#endif
#ifndef BR_K4L_EKEEP
#define BR_K4L_EKEEP 1   // 1: the coverage loop keeps the winner's three edge values, so that shading reads only its
                         // invD and face id from shared memory (the a, b, g words were ~25% of K4's shared wavefronts,
                         // half of them bank conflicts between the lanes' different winners)
#endif
#ifndef BR_K4L_R48
#define BR_K4L_R48 1   // 1: the grouped stage holds 48-B records (the 12 words the tests read) and a separate (invD, face)
                       // pair per slot: a 48-B stride spreads 8 consecutive slots over all 32 banks, so the stage's
                       // record stores are conflict-free (64-B records: 4-way conflicts, ~11% of K4's shared wavefronts)
#endif
#ifndef BR_K4L_WCLR
#define BR_K4L_WCLR 1   // 1: every warp clears its own footprint's counters (cnt, cntb, minz) right after its tests of a
#endif                  //    sub-frame -- NFP == NWARP, so warp w is their only reader -- and the group's third barrier goes
                        //    (C4 K4 5.634 -> 5.505 ms, C3 1.236 -> 1.203 ms, C5 217.8 -> 212.5 ms; parity green)
#ifndef BR_K4L_GTAU
#define BR_K4L_GTAU 0   // 1: the stage reads its sub-frame times from the schedule in global memory (in parallel with the
#endif                  //    bin entries) instead of S.taus, so no load sits between the chunk header and the group's barrier
                        //    (measured with WCLR on: C4 K4 5.50 -> 5.52 ms, C5 fwd 212.5 -> 213.8 ms, parity-green; kept off)
#ifndef BR_K4L_HPREF
#define BR_K4L_HPREF 0  // 1: the next chunk's header and bin offsets are copied to shared memory by cp.async while this chunk
#endif                  //    is staged (no registers held; made visible by the stage's barrier): one L2 round trip less per chunk
                        //    (measured: C4 K4 5.51 -> 5.98 ms, C3 1.21 -> 1.32 ms, C5 fwd 212.5 -> 231.1 ms; 16 B more spills and a
                        //    cp.async commit / wait per group; parity-green; kept off)
#ifndef BR_K4L_CULL
#define BR_K4L_CULL 2   // 2: faces turned away from the camera in a second list per footprint, tested last, the whole
                        // list skipped when every pixel's winner is nearer than the list's lowest depth; 0: one list
#endif                  //    (measured slower in this kernel: C4 K4 6.86 -> 7.17 ms)

#ifdef BR_K4L_STATS   // diagnostics build (tools/k4l_stats.py): counters in the workspace's status block
#define K4L_STAT(t_, i_, v_) atomicAdd(reinterpret_cast<unsigned long long *>((t_).status) + (i_), (unsigned long long)(v_))
#else
#define K4L_STAT(t_, i_, v_) ((void)0)
#endif

#ifdef BR_CHECKED
__device__ int *g_status_dbg;   // the launch's status word, for the checks inside the staging helpers
#endif

struct __align__(16) LeanSmem {
    TauRec rec[SREC_F];
    union {
        struct {
            uint16_t list[NFP][SREC_F];         // per footprint: sub-frame l's reaching records (byte offsets into rec)
            int cnt[GMAX_F][NFP];               // ... at [l * n, l * n + cnt): faces turned towards the camera,
            int cntb[GMAX_F][NFP];              // and at [l * n + n - cntb, l * n + n): the others
            int minz[GMAX_F][NFP];              // lowest depth of the others over the footprint (float bits, >= 0)
            int ent[BR_K4L_SENT ? SREC_F : 1];  // the chunk's bin entries (face ids)
            int acc_pairs[BR_K4L_TWOPASS ? SREC_F : 1];   // box-accepted pairs: j | l << 9 | box << 13
            int nacc;
        } g;                                    // grouped path
        struct {
            uint32_t wm[NFP * (SREC_F / 32 + GMAX_F)];
            int sid[SREC_F];
        } b;                                    // per-sub-frame batch path (long bins, fallback)
    } u;
    float taus[GMAX_F];
    int wsum[NWARP];
    float2 uv[NT];                              // the thread's pixel (ul, vl), reloaded per sub-frame
    float4 acc[TW * TH];                        // per-pixel (r, g, b, a) sums over the sub-frames
    int pent[BR_K4L_PREF ? SREC_F : 1];         // the next chunk's bin entries, prefetched by cp.async
    struct __align__(8) NHdr { int b, s, k0, k1; long long o, o1; } nh[2];   // BR_K4L_HPREF: prefetched chunk headers
};
static_assert(SREC_F * 64 <= 65535, "list entries are 16-bit byte offsets");
static_assert(!BR_K4L_GTAU || (!BR_K4L_LAZY && !BR_K4L_TWOPASS && !BR_K4L_TPREF), "S.taus is not written with BR_K4L_GTAU");
static_assert(!BR_K4L_HPREF || (!BR_K4L_TPREF && !BR_K4L_NWIN && !BR_K4L_PREF), "one prefetch scheme at a time");
static_assert(!BR_K4L_WCLR || (NFP == NWARP && !BR_K4L_LAZY && !BR_K4L_TWOPASS && !BR_K4L_TPREF),
              "per-warp counter clears: one warp per footprint, S.taus and nacc untouched by the tests");
// BR_K4L_R48 view of the grouped path's record stage (the batch path keeps TauRec[SREC_F] in the same bytes):
// 48-B records [0, SREC_F) followed by the (invD, face id) pairs
constexpr int R48_BYTES = 48;
static_assert(SREC_F * (R48_BYTES + 8) <= SREC_F * (int)sizeof(TauRec), "the 48-B view fits the record stage");
static_assert(!(BR_K4L_R48 && (BR_K4L_LAZY || !BR_K4L_EKEEP || BR_STAGE_EARLY)),
              "the 48-B records need EKEEP shading, no lazy staging and the record written after the masks");
__device__ __forceinline__ float2 *r48_x(TauRec *rec) { return reinterpret_cast<float2 *>(reinterpret_cast<float4 *>(rec) + 3 * SREC_F); }
__device__ __forceinline__ const float2 *r48_x(const TauRec *rec)
{
    return reinterpret_cast<const float2 *>(reinterpret_cast<const float4 *>(rec) + 3 * SREC_F);
}

// Stage faces [0, n) of the bin at the ng sub-frames taus[0..ng): records rec[l * n + j] and, for every
// footprint a record reaches, its byte offset in that footprint's list of sub-frame l (cnt must be zero).
// Each warp takes candidate pairs 32 at a time, and the pairs whose per-tau box reaches the tile go
// to a warp queue; the full stage (record load, Horner, footprint masks) runs on 32 queued pairs at a
// time, so the box rejects (about half the pairs) leave no lanes idle in it.
// the (face, sub-frame) pair p's first words: face, record, box test at tau (false: not staged)
__device__ __forceinline__ bool pair_head(const BinCtx &bc, const int *ent, int p, float inv_ng, int ng, const float *taus,
                                          const TileCtx &tc, int W, int H, int F, int &j, int &l, const float4 *&r,
                                          float &D, int &x0, int &x1, int &y0, int &y1)
{
    j = div_small(p, inv_ng);
    l = p - j * ng;
    const int f = (BR_K4L_SENT || BR_K4L_PREF) ? ent[j] : __ldg(ent + j);   // generic load: ent may be in shared memory
    if ((unsigned)f >= (unsigned)F) {     // never expected: bins hold valid face ids
        atomicOr(bc.status, BLUR_ST_EINTERNAL);
        return false;
    }
    r = bc.rseg + (size_t)f * REC_F4;
    const float4 q6 = __ldg(r + 6);
    const float4 b0 = __ldg(r + 7), b1 = __ldg(r + 8);
    if (__float_as_int(q6.w) < 0) return false;               // skipped face (Q8, behind, bad index)
    const float tau = taus[l];
    D = __fmaf_rn(tau, __fmaf_rn(tau, q6.x, q6.y), q6.z);       // a1 t^2 + a2 t + a3
    if (!(fabsf(D) > EPS_D)) return false;
    return tile_pixels(box_lerp(tau, b0.x, b1.x), box_lerp(tau, b0.y, b1.y), box_lerp(tau, b0.z, b1.z),
                       box_lerp(tau, b0.w, b1.w), W, H, tc, x0, x1, y0, y1);
}

__device__ __forceinline__ void pair_stage_fr(const FaceRec &fr, int j, int l, int n, float tau, float D, int x0, int x1,
                                              int y0, int y1, const TileCtx &tc, TauRec *rec, uint16_t (*list)[SREC_F],
                                              int (*cnt)[NFP], int (*cntb)[NFP], float sF, int (*minz)[NFP],
                                              unsigned long long *nstage);

__device__ __forceinline__ void pair_stage(const float4 *r, int j, int l, int n, float tau, float D, int x0, int x1,
                                           int y0, int y1, const TileCtx &tc, TauRec *rec, uint16_t (*list)[SREC_F],
                                           int (*cnt)[NFP], int (*cntb)[NFP], float sF, int (*minz)[NFP],
                                           unsigned long long *nstage = nullptr)
{
    FaceRec fr;
    load_rec(r, fr);
    pair_stage_fr(fr, j, l, n, tau, D, x0, x1, y0, y1, tc, rec, list, cnt, cntb, sF, minz, nstage);
}

__device__ __forceinline__ void pair_stage_fr(const FaceRec &fr, int j, int l, int n, float tau, float D, int x0, int x1,
                                              int y0, int y1, const TileCtx &tc, TauRec *rec, uint16_t (*list)[SREC_F],
                                              int (*cnt)[NFP], int (*cntb)[NFP], float sF, int (*minz)[NFP],
                                              unsigned long long *nstage)
{
    const bool back = BR_K4L_CULL && D * sF < 0.f;   // turned away from the camera (sF: mesh orientation)
#if BR_K4L_R48
    const int slot = l * n + j;
    float4 *d48 = reinterpret_cast<float4 *>(rec) + 3 * slot;   // the slot's 48-B record + (invD, face)
    const uint32_t fm = (BR_K4L_BACKBOX && back)
                            ? stage_tau<true, true, true>(fr, tau, D, x0, x1, y0, y1, tc, rec[0], d48, r48_x(rec) + slot)
                            : stage_tau<true, false, true>(fr, tau, D, x0, x1, y0, y1, tc, rec[0], d48, r48_x(rec) + slot);
    const uint16_t off = (uint16_t)(slot * R48_BYTES);
#else
    // the faces turned away are mostly skipped with their whole list: their footprints from the box alone
    const uint32_t fm = (BR_K4L_BACKBOX && back) ? stage_tau<true, true>(fr, tau, D, x0, x1, y0, y1, tc, rec[l * n + j])
                                                 : stage_tau<true>(fr, tau, D, x0, x1, y0, y1, tc, rec[l * n + j]);
    const uint16_t off = (uint16_t)((l * n + j) * (int)sizeof(TauRec));
#endif
    if (nstage) *nstage += fm != 0u;
    if (!back) {
        for (uint32_t m = fm; m; m &= m - 1) {
            const int w = __ffs(m) - 1;
            const int q = atomicAdd(&cnt[l][w], 1);
            BR_CHECK(q < n && l * n + q < SREC_F && w < NFP, g_status_dbg);
            list[w][l * n + q] = off;
        }
        return;
    }
#if BR_K4L_R48
    const float4 z48 = d48[2];   // (g2, az, bz, cz)
    const float az = z48.y, bz = z48.z, cz = z48.w;
#else
    const TauRec &R = rec[l * n + j];
    const float az = R.az, bz = R.bz, cz = R.cz;
#endif
    for (uint32_t m = fm; m; m &= m - 1) {
        const int w = __ffs(m) - 1;
        const int q = atomicAdd(&cntb[l][w], 1);
        BR_CHECK(q < n && l * n + n - 1 - q >= l * n && l * n + n - 1 < SREC_F && w < NFP, g_status_dbg);
        list[w][l * n + n - 1 - q] = off;
        if (BR_K4L_CULL == 2) {
            // the depth plane fma(az, ul, fma(bz, vl, cz)) is monotone in ul and vl: its minimum over the
            // footprint's pixel centres is its value at one corner (the lanes' own ul, vl values)
            const int wx = w & 1, wy = w >> 1;
            const float u = (float)((az > 0.f ? 0 : 7) + wx * FPW - TW / 2) * tc.sx;
            const float v = (float)(TH / 2 - wy * 4 - (bz > 0.f ? 3 : 0)) * tc.sy;
            const float zm = fmaxf(__fmaf_rn(az, u, __fmaf_rn(bz, v, cz)), 0.f);   // NaN -> 0 (no skip)
            atomicMin(&minz[l][w], __float_as_int(zm));
        }
    }
}

// Stage faces [0, n) of the bin (face ids ent[] in shared memory) at the ng sub-frames taus[0..ng): records
// rec[l * n + j] and, for every footprint a record reaches, its byte offset in that footprint's list of
// sub-frame l (counters must be zero).  A thread takes two pairs at a time and requests both pairs' first
// record words before testing either (the stage is a chain of L2 round trips: fewer of them per group).
__device__ __forceinline__ void stage_group_list(const BinCtx &bc, const int *ent, int n, const float *taus, int ng,
                                                 const TileCtx &tc, int W, int H, int F, TauRec *rec,
                                                 uint16_t (*list)[SREC_F], int (*cnt)[NFP], int (*cntb)[NFP], float sF,
                                                 int (*minz)[NFP], unsigned long long *nstage = nullptr)
{
    const int npair = n * ng;
    const float inv_ng = BR_K4L_MASKBF ? __frcp_rn((float)ng) : 1.0f / (float)ng;
#if BR_K4L_UNIT
    // units of (face j, block of kb consecutive sub-frames), at most one per thread: the face's whole record is
    // requested at once and evaluated at each sub-frame of the block (one L2 round trip per unit instead of two
    // per pair)
    const int kb = (npair + NT - 1) / NT, nb = (ng + kb - 1) / kb, nunit = n * nb;
    const float inv_nb = 1.0f / (float)nb;
    for (int u = threadIdx.x; u < nunit; u += NT) {
        const int j = div_small(u, inv_nb), lb = u - j * nb;
        const int f = (BR_K4L_SENT || BR_K4L_PREF) ? ent[j] : __ldg(ent + j);   // generic load: ent may be in shared memory
        if ((unsigned)f >= (unsigned)F) {     // never expected: bins hold valid face ids
            atomicOr(bc.status, BLUR_ST_EINTERNAL);
            continue;
        }
        FaceRec fr;
        load_rec(bc.rseg + (size_t)f * REC_F4, fr);
        if (__float_as_int(fr.q[6].w) < 0) continue;          // skipped face (Q8, behind, bad index)
        const int l1 = min(ng, lb * kb + kb);
        for (int l = lb * kb; l < l1; ++l) {
            const float tau = taus[l];
            const float D = __fmaf_rn(tau, __fmaf_rn(tau, fr.q[6].x, fr.q[6].y), fr.q[6].z);   // a1 t^2 + a2 t + a3
            if (!(fabsf(D) > EPS_D)) continue;
            int x0, x1, y0, y1;
            if (!tile_pixels(box_lerp(tau, fr.q[7].x, fr.q[8].x), box_lerp(tau, fr.q[7].y, fr.q[8].y),
                             box_lerp(tau, fr.q[7].z, fr.q[8].z), box_lerp(tau, fr.q[7].w, fr.q[8].w), W, H, tc, x0, x1, y0,
                             y1))
                continue;
            pair_stage_fr(fr, j, l, n, tau, D, x0, x1, y0, y1, tc, rec, list, cnt, cntb, sF, minz, nstage);
        }
    }
#elif BR_K4L_PAIR2
    for (int p0 = threadIdx.x; p0 < npair; p0 += 2 * NT) {
        const int p1 = p0 + NT;
        int ja, la, jb = 0, lb = 0, xa0, xa1, ya0, ya1, xb0 = 0, xb1 = 0, yb0 = 0, yb1 = 0;
        const float4 *ra, *rb = nullptr;
        float Da, Db = 0.f;
        const bool oka = pair_head(bc, ent, p0, inv_ng, ng, taus, tc, W, H, F, ja, la, ra, Da, xa0, xa1, ya0, ya1);
        const bool okb = p1 < npair && pair_head(bc, ent, p1, inv_ng, ng, taus, tc, W, H, F, jb, lb, rb, Db, xb0, xb1, yb0, yb1);
        if (oka) pair_stage(ra, ja, la, n, taus[la], Da, xa0, xa1, ya0, ya1, tc, rec, list, cnt, cntb, sF, minz);
        if (okb) pair_stage(rb, jb, lb, n, taus[lb], Db, xb0, xb1, yb0, yb1, tc, rec, list, cnt, cntb, sF, minz);
    }
#elif BR_K4L_ONELOAD
    // the whole record requested at once (one L2 round trip after the bin entry instead of two), also for the
    // pairs the box test then rejects
    for (int p = threadIdx.x; p < npair; p += NT) {
        const int j = div_small(p, inv_ng), l = p - j * ng;
        const int f = (BR_K4L_SENT || BR_K4L_PREF) ? ent[j] : __ldg(ent + j);
        if ((unsigned)f >= (unsigned)F) {
            atomicOr(bc.status, BLUR_ST_EINTERNAL);
            continue;
        }
        FaceRec fr;
        load_rec(bc.rseg + (size_t)f * REC_F4, fr);
        if (__float_as_int(fr.q[6].w) < 0) continue;                   // skipped face (Q8, behind, bad index)
        const float tau = taus[l];
        const float D = __fmaf_rn(tau, __fmaf_rn(tau, fr.q[6].x, fr.q[6].y), fr.q[6].z);
        if (!(fabsf(D) > EPS_D)) continue;
        int x0, x1, y0, y1;
        if (!tile_pixels(box_lerp(tau, fr.q[7].x, fr.q[8].x), box_lerp(tau, fr.q[7].y, fr.q[8].y),
                         box_lerp(tau, fr.q[7].z, fr.q[8].z), box_lerp(tau, fr.q[7].w, fr.q[8].w), W, H, tc, x0, x1, y0, y1))
            continue;
        pair_stage_fr(fr, j, l, n, tau, D, x0, x1, y0, y1, tc, rec, list, cnt, cntb, sF, minz, nstage);
    }
#else
    for (int p = threadIdx.x; p < npair; p += NT) {
        int j, l, x0, x1, y0, y1;
        const float4 *r;
        float D;
        if (pair_head(bc, ent, p, inv_ng, ng, taus, tc, W, H, F, j, l, r, D, x0, x1, y0, y1)
#ifdef BR_EXP_NOBACK
            && !(D * sF < 0.f)   // timing experiment only: faces turned away are never staged (not exact)
#endif
            ) {
#if BR_K4L_LAZY
            if (D * sF < 0.f) {   // turned away: only its depth bound and box footprints now (staged if needed)
                const float4 z0 = __ldg(r + 9), z1 = __ldg(r + 10);
                const float tau = taus[l];
                const float zlo = fminf(fminf(__fmaf_rn(tau, z1.x - z0.x, z0.x), __fmaf_rn(tau, z1.y - z0.y, z0.y)),
                                        __fmaf_rn(tau, z1.z - z0.z, z0.z));
                // the face's depth at any of its points is a convex combination of its corners' (Q6): >= zlo
                const int zb = __float_as_int(fmaxf(zlo, 0.f));   // NaN -> 0: never skips
                for (int wy = y0 >> 2; wy <= (y1 >> 2); ++wy)
                    for (int wx = x0 >> 3; wx <= (x1 >> 3); ++wx) {
                        const int w = wy * 2 + wx;
                        const int q = atomicAdd(&cntb[l][w], 1);
                        BR_CHECK(q < n && l * n + n - 1 < SREC_F, g_status_dbg);
                        list[w][l * n + n - 1 - q] = (uint16_t)j;   // the bin slot (not a record offset)
                        atomicMin(&minz[l][w], zb);
                    }
                continue;
            }
#endif
#ifdef BR_K4L_STATS
            unsigned long long ns = 0;
            pair_stage(r, j, l, n, taus[l], D, x0, x1, y0, y1, tc, rec, list, cnt, cntb, sF, minz, &ns);
            atomicAdd(reinterpret_cast<unsigned long long *>(bc.status) + 21, 1ull);
            if (ns) atomicAdd(reinterpret_cast<unsigned long long *>(bc.status) + (D * sF < 0.f ? 23 : 22), 1ull);
#else
            pair_stage(r, j, l, n, taus[l], D, x0, x1, y0, y1, tc, rec, list, cnt, cntb, sF, minz, nstage);
#endif
        }
    }
#endif
}

// Two passes: the box tests of all the group's pairs, the accepted ones compacted into apairs (warp-aggregated
// slots), a barrier, then the full stage over the accepted pairs -- every lane of the stage has a pair (about
// half the pairs miss the tile at their sub-frame).  nacc must be zero on entry; it is left nonzero.
__device__ __forceinline__ void stage_group_2pass(const BinCtx &bc, const int *ent, int n, const float *taus, int ng,
                                                  const TileCtx &tc, int W, int H, int F, TauRec *rec,
                                                  uint16_t (*list)[SREC_F], int (*cnt)[NFP], int (*cntb)[NFP], float sF,
                                                  int (*minz)[NFP], int *apairs, int *nacc)
{
    const int npair = n * ng, lane = threadIdx.x & 31;
    const float inv_ng = 1.0f / (float)ng;
    for (int p0 = threadIdx.x - lane; p0 < npair; p0 += NT) {   // warp-uniform trip count
        const int p = p0 + lane;
        int j = 0, l = 0, x0 = 0, x1 = 0, y0 = 0, y1 = 0;
        const float4 *r;
        float D;
        const bool ok = p < npair && pair_head(bc, ent, p, inv_ng, ng, taus, tc, W, H, F, j, l, r, D, x0, x1, y0, y1);
        const unsigned m = __ballot_sync(0xffffffffu, ok);
        int base = 0;
        if (lane == 0 && m) base = atomicAdd(nacc, __popc(m));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (ok) apairs[base + __popc(m & ((1u << lane) - 1u))] = j | (l << 9) | (x0 << 13) | (x1 << 17) | (y0 << 21) | (y1 << 25);
    }
    __syncthreads();
    const int na = *nacc;
    for (int i = threadIdx.x; i < na; i += NT) {
        const int code = apairs[i];
        const int j = code & 0x1FF, l = (code >> 9) & 0xF;
        const int f = (BR_K4L_SENT || BR_K4L_PREF) ? ent[j] : __ldg(ent + j);   // generic load: ent may be in shared memory
        const float4 *r = bc.rseg + (size_t)f * REC_F4;
        const float tau = taus[l];
        const float4 q6 = __ldg(r + 6);
        const float D = __fmaf_rn(tau, __fmaf_rn(tau, q6.x, q6.y), q6.z);
        pair_stage(r, j, l, n, tau, D, (code >> 13) & 0xF, (code >> 17) & 0xF, (code >> 21) & 0xF, (code >> 25) & 0xF, tc,
                   rec, list, cnt, cntb, sF, minz);
    }
}

#if BR_K4L_LAZY
// Lazily staged faces turned away from the camera: the warp stages the back list entries [i0, i1) of its
// footprint itself, 32 at a time (lane i: the face's record at tau for this tile, rec_at), and every lane tests
// them against its pixel with the values broadcast by shuffles -- the same TauRec, the same tests as the staged
// path (bit-identical), without a CTA barrier.  TIE: the Q7 re-run, comparing (depth, face index).
template <bool TIE, bool CENSUS>
__device__ __forceinline__ void lazy_back(const uint16_t *lst, int i0, int i1, const int *ent, const float4 *rseg, int F,
                                          int *status, float tau, const TileCtx &tc, float ul, float vl, int lane,
                                          float &zbest, int &eoff, float &tief, int &fbest, bool inimg,
                                          unsigned long long &c_cov, unsigned long long &c_test)
{
    for (int b0 = i0; b0 < i1; b0 += 32) {
        const int i = b0 + lane;
        TauRec R;
        R.a[0] = R.a[1] = R.a[2] = 0.f; R.b[0] = R.b[1] = R.b[2] = 0.f;
        R.g[0] = R.g[1] = R.g[2] = -1.f;   // no record: never covers
        R.az = R.bz = R.cz = 0.f;
        R.fid = 0x7fffffff;
        int jj = 0;
        if (i < i1) {
            jj = lst[i];
            const int f = (BR_K4L_SENT || BR_K4L_PREF) ? ent[jj] : __ldg(ent + jj);
            if ((unsigned)f < (unsigned)F) {
                FaceRec fr;
                load_rec(rseg + (size_t)f * REC_F4, fr);
                const float D = __fmaf_rn(tau, __fmaf_rn(tau, fr.q[6].x, fr.q[6].y), fr.q[6].z);
                if (__float_as_int(fr.q[6].w) >= 0 && fabsf(D) > EPS_D) rec_at(fr, tau, D, tc, R);
            } else {
                atomicOr(status, BLUR_ST_EINTERNAL);
            }
        }
        const int cnt = min(32, i1 - b0);
        for (int sl = 0; sl < cnt; ++sl) {
            const float a0 = __shfl_sync(0xffffffffu, R.a[0], sl), a1 = __shfl_sync(0xffffffffu, R.a[1], sl);
            const float a2 = __shfl_sync(0xffffffffu, R.a[2], sl), b0v = __shfl_sync(0xffffffffu, R.b[0], sl);
            const float b1 = __shfl_sync(0xffffffffu, R.b[1], sl), b2 = __shfl_sync(0xffffffffu, R.b[2], sl);
            const float g0 = __shfl_sync(0xffffffffu, R.g[0], sl), g1 = __shfl_sync(0xffffffffu, R.g[1], sl);
            const float g2 = __shfl_sync(0xffffffffu, R.g[2], sl), az = __shfl_sync(0xffffffffu, R.az, sl);
            const float bz = __shfl_sync(0xffffffffu, R.bz, sl), cz = __shfl_sync(0xffffffffu, R.cz, sl);
            const int js = __shfl_sync(0xffffffffu, jj, sl);
            const float e0 = edge_eval(a0, b0v, g0, ul, vl);
            const float e1 = edge_eval(a1, b1, g1, ul, vl);
            const float e2 = edge_eval(a2, b2, g2, ul, vl);
            const float z = __fmaf_rn(az, ul, __fmaf_rn(bz, vl, cz));
            const float emin = fminf(fminf(e0, e1), e2);
            if (CENSUS && inimg) { c_test++; c_cov += emin >= 0.f; }
            if (!TIE) {
                tief = (emin >= 0.f && z == zbest) ? 1.f : tief;
                if (emin >= 0.f && z < zbest) { zbest = z; eoff = 0x10000 | js; }
            } else {
                const int fs = __shfl_sync(0xffffffffu, R.fid, sl);
                if (emin >= 0.f && z <= zbest && (z < zbest || fs < fbest)) { zbest = z; eoff = 0x10000 | js; fbest = fs; }
            }
        }
    }
}
#endif

template <bool COV, bool CENSUS = false>
__global__ void __launch_bounds__(NT, BR_K4_MINB) k4l_raster_fwd(Tables t, float *__restrict__ out, int *__restrict__ ids,
                                                                int ids_k, unsigned long long *census = nullptr)
{
    static_assert(!BR_HALF, "the lean forward uses the warps' 8x4 footprints");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    LeanSmem &S = *reinterpret_cast<LeanSmem *>(smem_raw);
    const int b = blockIdx.y, tile = blockIdx.x;
    const ImgInfo &im = t.imgs[b];
    const int N = im.N, c_begin = im.chunk_begin, c_end = im.chunk_end, sched_off = im.sched_off;
    const long long rec_off = im.rec_off;
    TileCtx tc;
    tile_ctx(t, tile, tc);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int lx = (warp & 1) * 8 + (lane & 7), ly = (warp >> 1) * 4 + (lane >> 3);
    const int px = tc.px0 + lx, py = tc.py0 + ly;
    const bool inimg = px < t.W && py < t.H;
    const float ul = (float)(lx - TW / 2) * tc.sx;
    const float vl = (float)(TH / 2 - ly) * tc.sy;
    const int myp = ly * TW + lx;
    const size_t pix = ((size_t)b * t.H + py) * t.W + px;
    S.acc[myp] = make_float4(0.f, 0.f, 0.f, 0.f);
    S.uv[threadIdx.x] = make_float2(ul, vl);
    for (int i = threadIdx.x; i < GMAX_F * NFP; i += NT) {
        (&S.u.g.cnt[0][0])[i] = 0; (&S.u.g.cntb[0][0])[i] = 0; (&S.u.g.minz[0][0])[i] = 0x7f800000;
    }
    if (threadIdx.x == 0) S.u.g.nacc = 0;
    unsigned long long dz = 0, c_cov = 0, c_test = 0, c_shade = 0, c_stage = 0;   // census (CENSUS builds)
    const double orient = *t.orient;
    const float sF = orient > 0.0 ? 1.f : orient < 0.0 ? -1.f : 0.f;
    int pref_c = -1;   // chunk whose bin entries were prefetched into S.pent (BR_K4L_PREF)
#if BR_K4L_HPREF
    int hp_par = 0;        // S.nh[hp_par] holds this chunk's header when hp_ok (block-uniform)
    bool hp_ok = false;
#endif

#if BR_K4L_TPREF
    // software pipeline over the chunks: chunk c + splits's header and bin offsets are loaded at the top of
    // chunk c; the taus of the next group are loaded after the stage and stored to S.taus after the tests
    int tau_k = -1;   // S.taus holds the taus of sub-frames tau_k.. (when >= 0)
    Chunk chn;
    long long on = 0, on1 = 0;
    if (c_begin + (int)blockIdx.z < c_end) {
        const int c0 = c_begin + (int)blockIdx.z;
        chn = t.chunks[c0];
        on = t.off[(size_t)c0 * t.T + tile];
        on1 = t.off[(size_t)c0 * t.T + tile + 1];
    }
#endif
#if BR_K4L_NWIN && !BR_K4L_TPREF
    int nwin = 0;   // lane j: the bin size of the CTA's chunk (window start + j)
    for (int c = c_begin + (int)blockIdx.z, jc = 0; c < c_end; c += t.splits, ++jc) {
        if ((jc & 31) == 0) {
            const int cc = c + lane * t.splits;
            nwin = 0;
            if (cc < c_end) {
                const size_t b2 = (size_t)cc * t.T + tile;
                nwin = (int)(t.off[b2 + 1] - t.off[b2]);
            }
        }
        const int n = __shfl_sync(0xffffffffu, nwin, jc & 31);
        if (n == 0 && !ids && !COV) continue;   // nothing to render or record for this chunk
        const Chunk ch = t.chunks[c];
        const size_t bi = (size_t)c * t.T + tile;
        const long long o = t.off[bi];
#else
    for (int c = c_begin + (int)blockIdx.z; c < c_end; c += t.splits) {
#endif
#if BR_K4L_NWIN && !BR_K4L_TPREF
#elif BR_K4L_TPREF
        const Chunk ch = chn;
        const long long o = on;
        const int n = (int)(on1 - on);
        const bool has_next = c + t.splits < c_end;
        if (has_next) {
            const size_t bi2 = (size_t)(c + t.splits) * t.T + tile;
            chn = t.chunks[c + t.splits];
            on = t.off[bi2];
            on1 = t.off[bi2 + 1];
        }
#elif BR_K4L_HPREF
        Chunk ch;
        long long o;
        int n;
        if (hp_ok) {   // copied to shared memory while the previous chunk was staged
            const LeanSmem::NHdr &h = S.nh[hp_par];
            ch.s = h.s; ch.k0 = h.k0; ch.k1 = h.k1;
            o = h.o;
            n = (int)(h.o1 - o);
        } else {
            ch = t.chunks[c];
            const size_t bi = (size_t)c * t.T + tile;
            o = t.off[bi];
            n = (int)(t.off[bi + 1] - o);
        }
#else
        const Chunk ch = t.chunks[c];
        const size_t bi = (size_t)c * t.T + tile;
        const long long o = t.off[bi];
        const int n = (int)(t.off[bi + 1] - o);
#endif
        if (n == 0) {
            if (ids && inimg && ids_k >= ch.k0 && ids_k < ch.k1) ids[pix] = -1;
            if (COV) {
                const unsigned m = __ballot_sync(0xffffffffu, !inimg);
                if (lane == 0)
                    for (int k = ch.k0; k < ch.k1; ++k) t.covbits[cov_word(t, im, k, tile) + warp] = m;
            }
#if BR_K4L_HPREF
            hp_ok = false;   // no barrier in this chunk: the next one reads its header from global memory
#endif
            continue;
        }
#if BR_K4L_HPREF
        // the next chunk's header into the other buffer: its last readers were two barriers ago at least; the copies
        // are waited for before this chunk's barriers (wait_prior below), which make them visible to the CTA
        if (c + t.splits < c_end) {
            if (threadIdx.x < 4) {
                const int c2 = c + t.splits;
                const long long *src = threadIdx.x < 2 ? reinterpret_cast<const long long *>(t.chunks + c2) + threadIdx.x
                                                       : t.off + ((size_t)c2 * t.T + tile) + (threadIdx.x - 2);
                __pipeline_memcpy_async(reinterpret_cast<long long *>(&S.nh[hp_par ^ 1]) + threadIdx.x, src, 8);
            }
            __pipeline_commit();
            hp_par ^= 1;
            hp_ok = true;
        } else {
            hp_ok = false;
        }
#endif
        BinCtx bc;
        bc.status = t.status;
        bc.rseg = t.rec + (size_t)(rec_off + (long long)ch.s * t.F) * REC_F4;
        bc.key0 = nullptr;
        bc.key1 = nullptr;
        bc.fcol = t.fcol;
        bc.ent = t.entries + o;
        bc.n = n;
        bc.fb = o + n > t.cap;
        if (!bc.fb && n <= SREC_F) {
            const int Gs = BR_K4L_GRP >= SREC_F ? min(GMAX_F, group_div(SREC_F, n))
                                                : max(1, min(GMAX_F, group_div(BR_K4L_GRP, n)));
            uint16_t *vis_out = n <= VIS_MAXN ? t.vis : nullptr;
#if BR_K4L_SENT
            __syncthreads();   // the previous chunk's entries are consumed
            for (int j = threadIdx.x; j < n; j += NT) S.u.g.ent[j] = __ldg(bc.ent + j);
            const int *ents = S.u.g.ent;
#else
            const int *ents = (BR_K4L_PREF && pref_c == c) ? S.pent : bc.ent;
#endif
            for (int kg = ch.k0; kg < ch.k1; kg += Gs) {
                const int ng = min(Gs, ch.k1 - kg);
#if BR_K4L_TPREF
                if (tau_k != kg && threadIdx.x < ng) S.taus[threadIdx.x] = t.sched_tau[sched_off + kg + threadIdx.x];
#elif !BR_K4L_GTAU
                if (threadIdx.x < ng) S.taus[threadIdx.x] = t.sched_tau[sched_off + kg + threadIdx.x];
#endif
#if BR_K4L_PREF
                __pipeline_wait_prior(0);   // this thread's prefetched entries have landed
#endif
                __syncthreads();   // taus written; the previous group's lists and counters are consumed
#if BR_K4L_TWOPASS
                stage_group_2pass(bc, ents, n, S.taus, ng, tc, t.W, t.H, t.F, S.rec, S.u.g.list, S.u.g.cnt, S.u.g.cntb, sF,
                                  S.u.g.minz, S.u.g.acc_pairs, &S.u.g.nacc);
#elif !defined(BR_EXP_NOSTAGE)
                stage_group_list(bc, ents, n, BR_K4L_GTAU ? t.sched_tau + sched_off + kg : S.taus, ng, tc, t.W, t.H, t.F, S.rec,
                                 S.u.g.list, S.u.g.cnt, S.u.g.cntb, sF, S.u.g.minz, CENSUS ? &c_stage : nullptr);
#endif
#if BR_K4L_HPREF
                __pipeline_wait_prior(0);   // the next chunk's header has landed (threads 0-3; no-op otherwise)
#endif
                __syncthreads();
                if (threadIdx.x == 0) { K4L_STAT(t, 20, n * ng); K4L_STAT(t, 29, 1); }
#if BR_K4L_TPREF && !BR_K4L_LAZY
                // the next group's taus (this chunk's next group, else the next chunk's first), requested now and
                // stored after the tests (the tests do not read S.taus); taus past the image's N are not read
                const int k_nx = kg + Gs < ch.k1 ? kg + Gs : (has_next ? chn.k0 : -1);
                float tau_nx = 0.f;
                if (k_nx >= 0 && threadIdx.x < GMAX_F && k_nx + (int)threadIdx.x < N)
                    tau_nx = t.sched_tau[sched_off + k_nx + threadIdx.x];
#endif
#if BR_K4L_PREF
                if (kg + Gs >= ch.k1) {   // last group of the chunk: bring the next chunk's bin entries in during the tests
                    pref_c = -1;
                    const int c2 = c + t.splits;
                    if (c2 < c_end) {
                        const size_t bi2 = (size_t)c2 * t.T + tile;
                        const long long o2 = t.off[bi2];
                        const int n2 = (int)(t.off[bi2 + 1] - o2);
                        if (n2 > 0 && n2 <= SREC_F && o2 + n2 <= t.cap) {
                            for (int j = threadIdx.x; j < n2; j += NT) __pipeline_memcpy_async(S.pent + j, t.entries + o2 + j, 4);
                            __pipeline_commit();
                            pref_c = c2;
                        }
                    }
                }
#endif
                uint16_t *vrow = vis_out ? vis_out + ((size_t)(im.cov_off + kg) * t.T + tile) * (TW * TH) + myp : nullptr;
                const int l_ids = (ids && inimg) ? ids_k - kg : -1;
                const uint16_t *lst = S.u.g.list[warp];
                const unsigned char *rbase = reinterpret_cast<const unsigned char *>(S.rec);
                for (int l = 0; l < ng; ++l, lst += n) {
                    const TauRec *rl = S.rec + l * n;
#ifdef BR_EXP_NOVIS
                    const int cn = 0, cb = 0;
#else
                    const int cn = S.u.g.cnt[l][warp], cb = S.u.g.cntb[l][warp];
#endif
                    BR_CHECK(cn + cb <= n && (l + 1) * n <= SREC_F, t.status);
                    const float2 uvp = S.uv[threadIdx.x];
                    const float ul = uvp.x, vl = uvp.y;
                    float zbest = __int_as_float(0x7f800000), tief = 0.f;
                    int eoff = -1;
                    bool backs = false;   // BR_K4L_LAZY: the back list was tested (staged by this warp)
#if BR_K4L_EKEEP && !BR_K4L_LAZY
                    float ew0 = 0.f, ew1 = 0.f, ew2 = 0.f;   // the winner's edge values at this pixel
#define EKEEP_SET(a, b, c) (ew0 = (a), ew1 = (b), ew2 = (c))
#else
#define EKEEP_SET(a, b, c) ((void)0)
#endif
#ifdef BR_K4L_STATS
                    if (lane == 0) {
                        K4L_STAT(t, 24, 1); K4L_STAT(t, 25, cn + cb > 0); K4L_STAT(t, 26, cn); K4L_STAT(t, 28, cb);
                    }
#endif
                    // coverage loop: begin (tools/update_traffic.py)
                    BR_UNROLL4 for (int i = 0; i < cn; ++i) {   // faces turned towards the camera
                        const int off = lst[i];
                        const float4 *rp = reinterpret_cast<const float4 *>(rbase + off);
                        const float4 q0 = rp[0], q1 = rp[1], q2 = rp[2];
                        const float e0 = edge_eval(q0.x, q0.w, q1.z, ul, vl);
                        const float e1 = edge_eval(q0.y, q1.x, q1.w, ul, vl);
                        const float e2 = edge_eval(q0.z, q1.y, q2.x, ul, vl);
                        const float z = __fmaf_rn(q2.y, ul, __fmaf_rn(q2.z, vl, q2.w));
                        const float emin = fminf(fminf(e0, e1), e2);
                        if (CENSUS && inimg) { c_test++; c_cov += emin >= 0.f; }
                        tief = (emin >= 0.f && z == zbest) ? 1.f : tief;
                        if (emin >= 0.f && z < zbest) { zbest = z; eoff = off; EKEEP_SET(e0, e1, e2); }
                    }
                    if (BR_K4L_CULL == 2 && cb) {   // the others, unless all of them are behind every pixel's winner
#if BR_K4L_MICRO
                        // depths are positive: the integer order of their bits is the float order (one REDUX; a NaN
                        // gives a NaN maximum, which never skips)
                        const float zmax = __int_as_float(__reduce_max_sync(0xffffffffu, __float_as_int(zbest)));
#else
                        float zmax = zbest;
#pragma unroll
                        for (int d = 16; d > 0; d >>= 1) zmax = fmaxf(zmax, __shfl_xor_sync(0xffffffffu, zmax, d));
#endif
                        // zmax = +inf unless every pixel of the footprint has a winner; each face of the list has
                        // its depth >= minz at every pixel of the footprint (staging, corner of the plane)
                        if (!(zmax < __int_as_float(S.u.g.minz[l][warp]))) {
#ifdef BR_K4L_STATS
                            if (lane == 0) K4L_STAT(t, 27, cb);
#endif
#if BR_K4L_LAZY
                            backs = true;
                            int fdum = 0;
                            lazy_back<false, CENSUS>(lst, n - cb, n, ents, bc.rseg, t.F, t.status, S.taus[l], tc, ul, vl, lane,
                                                     zbest, eoff, tief, fdum, inimg, c_cov, c_test);
#else
                            BR_UNROLL4 for (int i = n - cb; i < n; ++i) {
                                const int off = lst[i];
                                const float4 *rp = reinterpret_cast<const float4 *>(rbase + off);
                                const float4 q0 = rp[0], q1 = rp[1], q2 = rp[2];
                                const float e0 = edge_eval(q0.x, q0.w, q1.z, ul, vl);
                                const float e1 = edge_eval(q0.y, q1.x, q1.w, ul, vl);
                                const float e2 = edge_eval(q0.z, q1.y, q2.x, ul, vl);
                                const float z = __fmaf_rn(q2.y, ul, __fmaf_rn(q2.z, vl, q2.w));
                                const float emin = fminf(fminf(e0, e1), e2);
                                if (CENSUS && inimg) { c_test++; c_cov += emin >= 0.f; }
                                tief = (emin >= 0.f && z == zbest) ? 1.f : tief;
                                if (emin >= 0.f && z < zbest) { zbest = z; eoff = off; EKEEP_SET(e0, e1, e2); }
                            }
#endif
                        }
                    }
                    // coverage loop: end
#if BR_K4L_WCLR
                    __syncwarp();   // every lane has read this footprint's counters
                    if (lane == 0) { S.u.g.cnt[l][warp] = 0; S.u.g.cntb[l][warp] = 0; S.u.g.minz[l][warp] = 0x7f800000; }
#endif
                    if (__any_sync(0xffffffffu, tief != 0.f)) {   // exact depth tie in the warp: face indices decide (Q7)
                        zbest = __int_as_float(0x7f800000);
                        eoff = -1;
                        int fbest = 0x7fffffff;
#if BR_K4L_LAZY
                        // faces turned away tie only if their list was tested (a skipped list is strictly behind)
                        if (backs) lazy_back<true, false>(lst, n - cb, n, ents, bc.rseg, t.F, t.status, S.taus[l], tc, ul, vl,
                                                          lane, zbest, eoff, tief, fbest, inimg, c_cov, c_test);
                        for (int ii = 0; ii < cn; ++ii) {
#else
                        for (int ii = 0; ii < cn + cb; ++ii) {
#endif
                            const int off = lst[ii < cn ? ii : n - cb + (ii - cn)];
                            const float4 *rp = reinterpret_cast<const float4 *>(rbase + off);
                            const float4 q0 = rp[0], q1 = rp[1], q2 = rp[2];
                            const float e0 = edge_eval(q0.x, q0.w, q1.z, ul, vl);
                            const float e1 = edge_eval(q0.y, q1.x, q1.w, ul, vl);
                            const float e2 = edge_eval(q0.z, q1.y, q2.x, ul, vl);
                            const float z = __fmaf_rn(q2.y, ul, __fmaf_rn(q2.z, vl, q2.w));
                            if (fminf(fminf(e0, e1), e2) >= 0.f && z <= zbest) {
#if BR_K4L_R48
                                const int fj = __float_as_int(r48_x(S.rec)[off / R48_BYTES].y);
#else
                                const int fj = reinterpret_cast<const TauRec *>(rbase + off)->fid;
#endif
                                if (z < zbest || fj < fbest) { zbest = z; eoff = off; fbest = fj; EKEEP_SET(e0, e1, e2); }
                            }
                        }
                    }
#if BR_K4L_LAZY
                    const int ebest = eoff >= 0x10000 ? (eoff & 0xFFFF) : eoff >= 0 ? eoff / (int)sizeof(TauRec) - l * n : -1;
#elif BR_K4L_R48
                    const int ebest = eoff >= 0 ? eoff / R48_BYTES - l * n : -1;
#else
                    const int ebest = eoff >= 0 ? eoff / (int)sizeof(TauRec) - l * n : -1;
#endif
                    int fid = -1;
                    if (ebest >= 0) {
                        float pr, pg, pb;
#if BR_K4L_LAZY
                        if (eoff >= 0x10000) {   // a face turned away won: its record again (rare)
                            const int f = (BR_K4L_SENT || BR_K4L_PREF) ? ents[ebest] : __ldg(ents + ebest);
                            FaceRec fr;
                            load_rec(bc.rseg + (size_t)f * REC_F4, fr);
                            const float tau = S.taus[l];
                            TauRec R;
                            rec_at(fr, tau, __fmaf_rn(tau, __fmaf_rn(tau, fr.q[6].x, fr.q[6].y), fr.q[6].z), tc, R);
                            shade(R, t.fcol, ul, vl, pr, pg, pb);      // Eq.9
                            fid = R.fid;
                        } else
#endif
                        {
#if BR_K4L_EKEEP && !BR_K4L_LAZY
                            // Eq.9 with the winner's edge values from the tests: w_i = e_i / |D|, the same
                            // arithmetic as shade() (edge_eval(a_i, b_i, g_i) * invD)
#if BR_K4L_R48
                            const float2 idf = r48_x(S.rec)[l * n + ebest];   // invD, fid
#else
                            const float2 idf = *reinterpret_cast<const float2 *>(&rl[ebest].invD);   // invD, fid
#endif
                            fid = __float_as_int(idf.y);
                            const float w0 = ew0 * idf.x, w1 = ew1 * idf.x, w2 = ew2 * idf.x;
                            const float4 *fc = t.fcol + 3 * (size_t)fid;
                            const float4 c0 = __ldg(fc), c1 = __ldg(fc + 1), c2 = __ldg(fc + 2);
                            pr = __fmaf_rn(w0, c0.x, __fmaf_rn(w1, c0.w, w2 * c1.z));
                            pg = __fmaf_rn(w0, c0.y, __fmaf_rn(w1, c1.x, w2 * c1.w));
                            pb = __fmaf_rn(w0, c0.z, __fmaf_rn(w1, c1.y, w2 * c2.x));
#else
                            shade(rl[ebest], t.fcol, ul, vl, pr, pg, pb);      // Eq.9
                            fid = rl[ebest].fid;
#endif
                        }
                        float4 a = S.acc[myp];
                        a.x += pr; a.y += pg; a.z += pb; a.w += 1.f;
                        S.acc[myp] = a;
                        if (CENSUS && inimg) c_shade++;
                    }
                    if (l == l_ids) ids[pix] = fid;
                    if (vrow) {   // visibility cache for K6
#if BR_VIS_STREAM
                        __stcs(vrow, ebest >= 0 ? (unsigned short)ebest : (unsigned short)0xFFFF);   // evict-first: keep L2 for the records
#else
                        *vrow = ebest >= 0 ? (uint16_t)ebest : (uint16_t)0xFFFF;
#endif
                        vrow += (size_t)t.T * (TW * TH);
                    }
                    if (COV) {   // soft path: which pixels of the warp are covered at this sub-frame
                        const unsigned m = __ballot_sync(0xffffffffu, ebest >= 0 || !inimg);
                        if (lane == 0) t.covbits[cov_word(t, im, kg + l, tile) + warp] = m;
                    }
                }
#if BR_K4L_TPREF && !BR_K4L_LAZY
                if (k_nx >= 0 && threadIdx.x < GMAX_F) S.taus[threadIdx.x] = tau_nx;
                tau_k = k_nx;
#endif
#if !BR_K4L_WCLR
                __syncthreads();   // lists read: clear the counters of this group
                if (threadIdx.x < ng * NFP) {
                    (&S.u.g.cnt[0][0])[threadIdx.x] = 0; (&S.u.g.cntb[0][0])[threadIdx.x] = 0;
                    (&S.u.g.minz[0][0])[threadIdx.x] = 0x7f800000;
                }
                if (threadIdx.x == 0) S.u.g.nacc = 0;
#endif
            }
#undef EKEEP_SET
        } else {
            // per sub-frame, several batches (long bins) or the exact fallback scan (overflow): as k4_raster_fwd
#if BR_K4L_TPREF
            tau_k = -1;   // S.taus[0] is rewritten here
#endif
            for (int k = ch.k0; k < ch.k1; ++k) {
                const float tau = t.sched_tau[sched_off + k];
                float zbest = __int_as_float(0x7f800000);
                int ebest = -1, bfid = -1, fbest = 0x7fffffff;
                bool has = false;
                float pr = 0.f, pg = 0.f, pb = 0.f;
                int base = 0, fpos = 0;
                __syncthreads();
                if (threadIdx.x == 0) S.taus[0] = tau;
                while (true) {
                    const int nb = next_batch(bc, t.F, tau, tc, t.W, t.H, SREC_F, base, fpos, S.u.b.sid, S.wsum);
                    if (nb == 0) break;
                    const int nw = (nb + 31) >> 5;
                    clear_words(S.u.b.wm, NFP * nw);
                    __syncthreads();
                    stage_group<CENSUS, 0, true>(bc, nb, base, S.taus, 1, tc, t.W, t.H, t.F, S.u.b.sid, S.rec, nullptr, S.u.b.wm, c_stage);
                    __syncthreads();
                    vis_mask<CENSUS, 0>(S.rec, nullptr, S.u.b.wm + warp * nw, nw, base, ul, vl, zbest, ebest, fbest, c_cov, c_test, inimg);
                    if (ebest >= base) {   // winner changed in this batch: shade now (Eq.9)
                        shade(S.rec[ebest - base], t.fcol, ul, vl, pr, pg, pb);
                        has = true;
                        bfid = S.rec[ebest - base].fid;
                        fbest = bfid;      // ties against later batches compare face indices
                    }
                    base += nb;
                    __syncthreads();
                }
                if (CENSUS && has && inimg) c_shade++;
                if (has) {
                    float4 a = S.acc[myp];
                    a.x += pr; a.y += pg; a.z += pb; a.w += 1.f;
                    S.acc[myp] = a;
                }
                if (ids && inimg && k == ids_k) ids[pix] = has ? bfid : -1;
                if (COV) {
                    const unsigned m = __ballot_sync(0xffffffffu, has || !inimg);
                    if (lane == 0) t.covbits[cov_word(t, im, k, tile) + warp] = m;
                }
            }
#if BR_K4L_HPREF
            __pipeline_wait_prior(0);
#endif
            __syncthreads();   // the grouped path's counters share the batch path's shared memory
            for (int i = threadIdx.x; i < GMAX_F * NFP; i += NT) {
                (&S.u.g.cnt[0][0])[i] = 0; (&S.u.g.cntb[0][0])[i] = 0; (&S.u.g.minz[0][0])[i] = 0x7f800000;
            }
            if (threadIdx.x == 0) S.u.g.nacc = 0;
        }
    }
    if (inimg && out) {   // out == null: coverage-only pass (soft backward without a preceding forward)
        const float inv = 1.0f / (float)N;
        const float4 a = S.acc[myp];
        const float4 v = make_float4(a.x * inv, a.y * inv, a.z * inv, a.w * inv);
        if (t.splits == 1) reinterpret_cast<float4 *>(out)[pix] = v;
        else t.part[(size_t)blockIdx.z * ((size_t)t.B * t.H * t.W) + pix] = v;
    }
    if (CENSUS) {
        atomicAdd(census + 0, c_cov);
        atomicAdd(census + 1, c_shade);
        atomicAdd(census + 2, c_test);
        atomicAdd(census + 3, c_stage);
    }
}

template <bool COV, bool CENSUS = false>
static cudaError_t launch_fwd_lean(const Tables &t, float *out, int *ids, int ids_k, cudaStream_t st,
                                   unsigned long long *census = nullptr)
{
    dim3 grid(t.T, t.B, t.splits);
    const int smem = (int)sizeof(LeanSmem);
    cudaError_t e = cudaFuncSetAttribute(k4l_raster_fwd<COV, CENSUS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
#ifdef BR_CHECKED
    e = cudaMemcpyToSymbolAsync(g_status_dbg, &t.status, sizeof(int *), 0, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return e;
#endif
    k4l_raster_fwd<COV, CENSUS><<<grid, NT, smem, st>>>(t, out, ids, ids_k, census);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ super-grouped lean forward (measured A/B)
//
// k4s_raster_fwd: k4l_raster_fwd with super-groups.  The automatic chunks of fast motions hold 2-3 sub-frames, so
// a k4l group is one chunk: ~200 (face, sub-frame) pairs staged between two barriers, ~20 (sub-frame, footprint)
// visits, and a third barrier to clear the counters (C4: 4.4e5 groups per launch, barrier waits the top stall).
// Here a group takes consecutive chunks of this CTA's share of the tile, sub-frame slot by slot, while the
// records fit (SREC_F) and the slots GMAX_F: each slot L has its own record range [rb_L, rb_L + n_L) -- its
// chunk's bin at its sub-frame -- and its own footprint lists in the same index range (faces turned towards the
// camera from the start, the others from the end), so the stage, the tests, the tie rule (Q7), the list-level
// skip of the faces turned away and the shading (Eq.9) are exactly k4l's; only the grouping differs.  Long and
// overflowed bins flush the group and take k4l's per-sub-frame batch path.

struct SGSeg {             // one chunk's part of a super-group (block-uniform, shared memory)
    const int *ent;        // bin entries (face ids)
    const float4 *rseg;    // records of the chunk's (image, segment)
    int n, ng;             // bin length, sub-frame slots taken
    int pbase, lbase;      // first pair, first slot of this part
    int rbase;             // first record
};
constexpr int SG_MAXC = GMAX_F;

struct __align__(16) SGSmem {
    LeanSmem L;
    SGSeg seg[SG_MAXC];
    int slot_rb[GMAX_F];   // per slot: first record, bin length, absolute sub-frame, visibility cache on
    int slot_n[GMAX_F];
    int slot_k[GMAX_F];
    int slot_vis[GMAX_F];
};

static_assert(BR_K4L_PREF || BR_K4_MINB > 5 || sizeof(SGSmem) + 1024 <= 228 * 1024 / BR_K4_MINB, "k4s_raster_fwd: BR_K4_MINB CTAs per SM");

__device__ __forceinline__ void pair_stage_sg(const FaceRec &fr, int ri, int rb, int n, int L, float tau, float D, int x0,
                                              int x1, int y0, int y1, const TileCtx &tc, TauRec *rec,
                                              uint16_t (*list)[SREC_F], int (*cnt)[NFP], int (*cntb)[NFP], float sF,
                                              int (*minz)[NFP])
{
    const bool back = BR_K4L_CULL && D * sF < 0.f;
    const uint32_t fm = stage_tau<true>(fr, tau, D, x0, x1, y0, y1, tc, rec[ri]);
    const uint16_t off = (uint16_t)(ri * (int)sizeof(TauRec));
    if (!back) {
        for (uint32_t m = fm; m; m &= m - 1) {
            const int w = __ffs(m) - 1;
            const int q = atomicAdd(&cnt[L][w], 1);
            BR_CHECK(q < n && rb + q < SREC_F && L < GMAX_F, g_status_dbg);
            list[w][rb + q] = off;
        }
        return;
    }
    const TauRec &R = rec[ri];
    const float az = R.az, bz = R.bz, cz = R.cz;
    for (uint32_t m = fm; m; m &= m - 1) {
        const int w = __ffs(m) - 1;
        const int q = atomicAdd(&cntb[L][w], 1);
        BR_CHECK(q < n && rb + n - 1 < SREC_F && L < GMAX_F, g_status_dbg);
        list[w][rb + n - 1 - q] = off;
        if (BR_K4L_CULL == 2) {   // lowest depth of the plane over the footprint's pixel centres (k4l)
            const int wx = w & 1, wy = w >> 1;
            const float u = (float)((az > 0.f ? 0 : 7) + wx * FPW - TW / 2) * tc.sx;
            const float v = (float)(TH / 2 - wy * 4 - (bz > 0.f ? 3 : 0)) * tc.sy;
            const float zm = fmaxf(__fmaf_rn(az, u, __fmaf_rn(bz, v, cz)), 0.f);
            atomicMin(&minz[L][w], __float_as_int(zm));
        }
    }
}

template <bool COV>
__global__ void __launch_bounds__(NT, BR_K4_MINB) k4s_raster_fwd(Tables t, float *__restrict__ out, int *__restrict__ ids,
                                                                int ids_k)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SGSmem &SG = *reinterpret_cast<SGSmem *>(smem_raw);
    LeanSmem &S = SG.L;
    const int b = blockIdx.y, tile = blockIdx.x;
    const ImgInfo &im = t.imgs[b];
    const int N = im.N, c_end = im.chunk_end, sched_off = im.sched_off;
    const long long rec_off = im.rec_off;
    TileCtx tc;
    tile_ctx(t, tile, tc);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int lx = (warp & 1) * 8 + (lane & 7), ly = (warp >> 1) * 4 + (lane >> 3);
    const int px = tc.px0 + lx, py = tc.py0 + ly;
    const bool inimg = px < t.W && py < t.H;
    const float ul0 = (float)(lx - TW / 2) * tc.sx;
    const float vl0 = (float)(TH / 2 - ly) * tc.sy;
    const int myp = ly * TW + lx;
    const size_t pix = ((size_t)b * t.H + py) * t.W + px;
    S.acc[myp] = make_float4(0.f, 0.f, 0.f, 0.f);
    S.uv[threadIdx.x] = make_float2(ul0, vl0);
    for (int i = threadIdx.x; i < GMAX_F * NFP; i += NT) {
        (&S.u.g.cnt[0][0])[i] = 0; (&S.u.g.cntb[0][0])[i] = 0; (&S.u.g.minz[0][0])[i] = 0x7f800000;
    }
    unsigned long long c_stage = 0;
    const double orient = *t.orient;
    const float sF = orient > 0.0 ? 1.f : orient < 0.0 ? -1.f : 0.f;

    int c = im.chunk_begin + (int)blockIdx.z;   // next chunk of this CTA's share, and its next sub-frame
    int kc = c < c_end ? t.chunks[c].k0 : 0;
    while (c < c_end) {
        // ---- compose a super-group (every thread computes the same composition from the same words)
        int nseg = 0, P = 0, R = 0, NL = 0;
        bool batch_chunk = false;
        while (c < c_end) {
            const Chunk ch = t.chunks[c];
            const size_t bi = (size_t)c * t.T + tile;
            const long long o = t.off[bi];
            const int n = (int)(t.off[bi + 1] - o);
            if (n == 0) {   // nothing covers the tile: background at every sub-frame of the chunk
                if (ids && inimg && ids_k >= ch.k0 && ids_k < ch.k1) ids[pix] = -1;
                if (COV) {
                    const unsigned m = __ballot_sync(0xffffffffu, !inimg);
                    if (lane == 0)
                        for (int k = ch.k0; k < ch.k1; ++k) t.covbits[cov_word(t, im, k, tile) + warp] = m;
                }
                c += t.splits;
                kc = c < c_end ? t.chunks[c].k0 : 0;
                continue;
            }
            if (o + n > t.cap || n > SREC_F) {   // long or overflowed bin: after the pending group, alone
                batch_chunk = nseg == 0;
                break;
            }
            const int ng = min(min(ch.k1 - kc, GMAX_F - NL), (SREC_F - R) / n);
            if (ng <= 0) break;   // group full
            if (threadIdx.x == 0) {
                SGSeg &sg = SG.seg[nseg];
                sg.ent = t.entries + o;
                sg.rseg = t.rec + (size_t)(rec_off + (long long)ch.s * t.F) * REC_F4;
                sg.n = n; sg.ng = ng; sg.pbase = P; sg.lbase = NL; sg.rbase = R;
            }
            if (threadIdx.x < ng) {
                const int L = NL + threadIdx.x;
                S.taus[L] = t.sched_tau[sched_off + kc + threadIdx.x];
                SG.slot_rb[L] = R + threadIdx.x * n;
                SG.slot_n[L] = n;
                SG.slot_k[L] = kc + threadIdx.x;
                SG.slot_vis[L] = n <= VIS_MAXN;
            }
            ++nseg; P += n * ng; R += n * ng; NL += ng;
            kc += ng;
            if (kc >= ch.k1) {
                c += t.splits;
                kc = c < c_end ? t.chunks[c].k0 : 0;
            }
            if (NL >= GMAX_F) break;
        }
        if (nseg > 0) {
            __syncthreads();   // composition written; the previous group's lists and counters are consumed
            // ---- stage: pairs over the parts, part by part
            for (int p = threadIdx.x; p < P; p += NT) {
                int s = 0;
                while (s + 1 < nseg && SG.seg[s + 1].pbase <= p) ++s;
                const SGSeg &sg = SG.seg[s];
                const int pl = p - sg.pbase, ng = sg.ng, n = sg.n;
                const int j = div_small(pl, __frcp_rn((float)ng));
                const int l = pl - j * ng, L = sg.lbase + l;
                const int f = __ldg(sg.ent + j);
                if ((unsigned)f >= (unsigned)t.F) { atomicOr(t.status, BLUR_ST_EINTERNAL); continue; }
                const float4 *r = sg.rseg + (size_t)f * REC_F4;
                const float4 q6 = __ldg(r + 6);
                const float4 b0 = __ldg(r + 7), b1 = __ldg(r + 8);
                if (__float_as_int(q6.w) < 0) continue;   // skipped face (Q8, behind, bad index)
                const float tau = S.taus[L];
                const float D = __fmaf_rn(tau, __fmaf_rn(tau, q6.x, q6.y), q6.z);
                if (!(fabsf(D) > EPS_D)) continue;
                int x0, x1, y0, y1;
                if (!tile_pixels(box_lerp(tau, b0.x, b1.x), box_lerp(tau, b0.y, b1.y), box_lerp(tau, b0.z, b1.z),
                                 box_lerp(tau, b0.w, b1.w), t.W, t.H, tc, x0, x1, y0, y1))
                    continue;
                FaceRec fr;
                load_rec(r, fr);
                const int rb = sg.rbase + l * n;
                pair_stage_sg(fr, rb + j, rb, n, L, tau, D, x0, x1, y0, y1, tc, S.rec, S.u.g.list, S.u.g.cnt,
                              S.u.g.cntb, sF, S.u.g.minz);
            }
            __syncthreads();
            // ---- visibility and shading per slot (k4l's loop body)
            const unsigned char *rbase = reinterpret_cast<const unsigned char *>(S.rec);
            for (int L = 0; L < NL; ++L) {
                const int rb = SG.slot_rb[L], n = SG.slot_n[L], k = SG.slot_k[L];
                const uint16_t *lst = S.u.g.list[warp] + rb;
                const int cn = S.u.g.cnt[L][warp], cb = S.u.g.cntb[L][warp];
                BR_CHECK(cn + cb <= n && rb + n <= SREC_F, t.status);
                const float2 uvp = S.uv[threadIdx.x];
                const float ul = uvp.x, vl = uvp.y;
                float zbest = __int_as_float(0x7f800000), tief = 0.f;
                int eoff = -1;
                for (int i = 0; i < cn; ++i) {   // faces turned towards the camera
                    const int off = lst[i];
                    const float4 *rp = reinterpret_cast<const float4 *>(rbase + off);
                    const float4 q0 = rp[0], q1 = rp[1], q2 = rp[2];
                    const float e0 = edge_eval(q0.x, q0.w, q1.z, ul, vl);
                    const float e1 = edge_eval(q0.y, q1.x, q1.w, ul, vl);
                    const float e2 = edge_eval(q0.z, q1.y, q2.x, ul, vl);
                    const float z = __fmaf_rn(q2.y, ul, __fmaf_rn(q2.z, vl, q2.w));
                    const float emin = fminf(fminf(e0, e1), e2);
                    tief = (emin >= 0.f && z == zbest) ? 1.f : tief;
                    if (emin >= 0.f && z < zbest) { zbest = z; eoff = off; }
                }
                if (BR_K4L_CULL == 2 && cb) {   // the others, unless all of them are behind every pixel's winner
                    const float zmax = __int_as_float(__reduce_max_sync(0xffffffffu, __float_as_int(zbest)));
                    if (!(zmax < __int_as_float(S.u.g.minz[L][warp]))) {
                        for (int i = n - cb; i < n; ++i) {
                            const int off = lst[i];
                            const float4 *rp = reinterpret_cast<const float4 *>(rbase + off);
                            const float4 q0 = rp[0], q1 = rp[1], q2 = rp[2];
                            const float e0 = edge_eval(q0.x, q0.w, q1.z, ul, vl);
                            const float e1 = edge_eval(q0.y, q1.x, q1.w, ul, vl);
                            const float e2 = edge_eval(q0.z, q1.y, q2.x, ul, vl);
                            const float z = __fmaf_rn(q2.y, ul, __fmaf_rn(q2.z, vl, q2.w));
                            const float emin = fminf(fminf(e0, e1), e2);
                            tief = (emin >= 0.f && z == zbest) ? 1.f : tief;
                            if (emin >= 0.f && z < zbest) { zbest = z; eoff = off; }
                        }
                    }
                }
                if (__any_sync(0xffffffffu, tief != 0.f)) {   // exact depth tie in the warp: face indices decide (Q7)
                    zbest = __int_as_float(0x7f800000);
                    eoff = -1;
                    int fbest = 0x7fffffff;
                    for (int ii = 0; ii < cn + cb; ++ii) {
                        const int off = lst[ii < cn ? ii : n - cb + (ii - cn)];
                        const float4 *rp = reinterpret_cast<const float4 *>(rbase + off);
                        const float4 q0 = rp[0], q1 = rp[1], q2 = rp[2];
                        const float e0 = edge_eval(q0.x, q0.w, q1.z, ul, vl);
                        const float e1 = edge_eval(q0.y, q1.x, q1.w, ul, vl);
                        const float e2 = edge_eval(q0.z, q1.y, q2.x, ul, vl);
                        const float z = __fmaf_rn(q2.y, ul, __fmaf_rn(q2.z, vl, q2.w));
                        if (fminf(fminf(e0, e1), e2) >= 0.f && z <= zbest) {
                            const int fj = reinterpret_cast<const TauRec *>(rbase + off)->fid;
                            if (z < zbest || fj < fbest) { zbest = z; eoff = off; fbest = fj; }
                        }
                    }
                }
                const int eb = eoff >= 0 ? eoff / (int)sizeof(TauRec) : -1;   // record index
                int fid = -1;
                if (eb >= 0) {
                    float pr, pg, pbb;
                    shade(S.rec[eb], t.fcol, ul, vl, pr, pg, pbb);      // Eq.9
                    float4 a = S.acc[myp];
                    a.x += pr; a.y += pg; a.z += pbb; a.w += 1.f;
                    S.acc[myp] = a;
                    fid = S.rec[eb].fid;
                }
                if (ids && inimg && k == ids_k) ids[pix] = fid;
                if (t.vis && SG.slot_vis[L])   // visibility cache for K6: the winner's slot in its bin
                    t.vis[((size_t)(im.cov_off + k) * t.T + tile) * (TW * TH) + myp] =
                        eb >= 0 ? (uint16_t)(eb - rb) : (uint16_t)0xFFFF;
                if (COV) {
                    const unsigned m = __ballot_sync(0xffffffffu, eb >= 0 || !inimg);
                    if (lane == 0) t.covbits[cov_word(t, im, k, tile) + warp] = m;
                }
            }
            __syncthreads();   // lists read: clear the counters of this group
            if (threadIdx.x < NL * NFP) {
                (&S.u.g.cnt[0][0])[threadIdx.x] = 0; (&S.u.g.cntb[0][0])[threadIdx.x] = 0;
                (&S.u.g.minz[0][0])[threadIdx.x] = 0x7f800000;
            }
            continue;
        }
        if (!batch_chunk) continue;
        // ---- a long or overflowed bin: per sub-frame, several batches or the exact fallback scan (as k4l)
        {
            const Chunk ch = t.chunks[c];
            const size_t bi = (size_t)c * t.T + tile;
            const long long o = t.off[bi];
            BinCtx bc;
            bc.status = t.status;
            bc.rseg = t.rec + (size_t)(rec_off + (long long)ch.s * t.F) * REC_F4;
            bc.key0 = nullptr;
            bc.key1 = nullptr;
            bc.fcol = t.fcol;
            bc.ent = t.entries + o;
            bc.n = (int)(t.off[bi + 1] - o);
            bc.fb = o + bc.n > t.cap;
            const float ul = ul0, vl = vl0;
            unsigned long long c_cov = 0, c_test = 0;
            for (int k = ch.k0; k < ch.k1; ++k) {
                const float tau = t.sched_tau[sched_off + k];
                float zbest = __int_as_float(0x7f800000);
                int ebest = -1, bfid = -1, fbest = 0x7fffffff;
                bool has = false;
                float pr = 0.f, pg = 0.f, pbb = 0.f;
                int base = 0, fpos = 0;
                __syncthreads();
                if (threadIdx.x == 0) S.taus[0] = tau;
                while (true) {
                    const int nb = next_batch(bc, t.F, tau, tc, t.W, t.H, SREC_F, base, fpos, S.u.b.sid, S.wsum);
                    if (nb == 0) break;
                    const int nw = (nb + 31) >> 5;
                    clear_words(S.u.b.wm, NFP * nw);
                    __syncthreads();
                    stage_group<false, 0, true>(bc, nb, base, S.taus, 1, tc, t.W, t.H, t.F, S.u.b.sid, S.rec, nullptr,
                                                S.u.b.wm, c_stage);
                    __syncthreads();
                    vis_mask<false, 0>(S.rec, nullptr, S.u.b.wm + warp * nw, nw, base, ul, vl, zbest, ebest, fbest, c_cov,
                                       c_test, inimg);
                    if (ebest >= base) {   // winner changed in this batch: shade now (Eq.9)
                        shade(S.rec[ebest - base], t.fcol, ul, vl, pr, pg, pbb);
                        has = true;
                        bfid = S.rec[ebest - base].fid;
                        fbest = bfid;
                    }
                    base += nb;
                    __syncthreads();
                }
                if (has) {
                    float4 a = S.acc[myp];
                    a.x += pr; a.y += pg; a.z += pbb; a.w += 1.f;
                    S.acc[myp] = a;
                }
                if (ids && inimg && k == ids_k) ids[pix] = has ? bfid : -1;
                if (COV) {
                    const unsigned m = __ballot_sync(0xffffffffu, has || !inimg);
                    if (lane == 0) t.covbits[cov_word(t, im, k, tile) + warp] = m;
                }
            }
            __syncthreads();   // the grouped path's counters share the batch path's shared memory
            for (int i = threadIdx.x; i < GMAX_F * NFP; i += NT) {
                (&S.u.g.cnt[0][0])[i] = 0; (&S.u.g.cntb[0][0])[i] = 0; (&S.u.g.minz[0][0])[i] = 0x7f800000;
            }
            c += t.splits;
            kc = c < c_end ? t.chunks[c].k0 : 0;
        }
    }
    if (inimg && out) {   // out == null: coverage-only pass (soft backward without a preceding forward)
        const float inv = 1.0f / (float)N;
        const float4 a = S.acc[myp];
        const float4 v = make_float4(a.x * inv, a.y * inv, a.z * inv, a.w * inv);
        if (t.splits == 1) reinterpret_cast<float4 *>(out)[pix] = v;
        else t.part[(size_t)blockIdx.z * ((size_t)t.B * t.H * t.W) + pix] = v;
    }
}

template <bool COV>
static cudaError_t launch_fwd_sg(const Tables &t, float *out, int *ids, int ids_k, cudaStream_t st)
{
    dim3 grid(t.T, t.B, t.splits);
    const int smem = (int)sizeof(SGSmem);
    cudaError_t e = cudaFuncSetAttribute(k4s_raster_fwd<COV>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
#ifdef BR_CHECKED
    e = cudaMemcpyToSymbolAsync(g_status_dbg, &t.status, sizeof(int *), 0, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return e;
#endif
    k4s_raster_fwd<COV><<<grid, NT, smem, st>>>(t, out, ids, ids_k);
    return cudaGetLastError();
}

// BLURRAST_FWD=sg: the super-grouped k4s_raster_fwd instead of k4l_raster_fwd (A/B; measured slower: C4 K4 5.92 ->
// 6.34 ms, C3 1.26 -> 1.39 ms, parity-green)
static bool sg_fwd_on()
{
    const char *s = std::getenv("BLURRAST_FWD");
    return s && std::strcmp(s, "sg") == 0;
}

// ------------------------------------------------------------------ pipelined forward (fast solver)
//
// k4p_raster_fwd: K4 with warp specialisation.  Staging a group of (face, sub-frame) records is a chain
// of dependent L2 loads (bin entry -> record words -> record); in k4l_raster_fwd every warp of the CTA
// waits for it at a barrier before the footprint tests start (measured: with the tests removed,
// k4l still takes 55% of its time).  Here 4 producer warps stage group g+1 into one of two record
// buffers while the 8 consumer warps (one 8x4 footprint each) test and shade group g from the other;
// the hand-off is a pair of named barriers per buffer (FULL: producers arrive, consumers wait;
// EMPTY: consumers arrive, producers wait), so neither side waits for the other's latency.  The
// records, tests, tie rule (Q7) and shading (Eq.9) are those of k4l_raster_fwd; the producers also
// build the per-footprint record lists there (faces turned towards the camera first, BR_K4P_CULL).
// Long bins and overflowed bins go through the same pipeline as per-sub-frame batches.

#ifndef BR_KP_SREC
#define BR_KP_SREC 256
#endif
#ifndef BR_K4P_CULL
#define BR_K4P_CULL 1
#endif
#ifndef BR_KP_MINB
#define BR_KP_MINB 3
#endif
constexpr int KP_SREC = BR_KP_SREC;   // records per buffer
#ifndef BR_KP_NP
#define BR_KP_NP 128
#endif
constexpr int KP_NP = BR_KP_NP;       // producer threads (warps 8..)
constexpr int KP_NTH = NT + KP_NP;
static_assert(KP_SREC * 64 <= 65535 && VIS_MAXN <= KP_SREC, "list offsets are 16-bit; cached bins take the group path");
enum { KP_GROUP = 0, KP_BATCH = 1, KP_EMPTY = 2, KP_END = 3 };

struct KpDesc {
    int kind, n, ng, kg, k1, last;
};

struct __align__(16) KpSmem {
    TauRec rec[2][KP_SREC];
    uint16_t list[2][NFP][KP_SREC];          // per footprint: sub-frame l's records at [l*n, l*n + cnt) (towards
    int cnt[2][GMAX_F][NFP];                 // the camera) and [l*n + n - cntb, l*n + n) (the others); byte
    int cntb[2][GMAX_F][NFP];                // offsets into rec[b]
    KpDesc desc[2];
    float taus[2][GMAX_F];
    int sid[KP_SREC];                        // the chunk's bin face ids / an overflowed bin's batch (producers)
    float4 raw[KP_NP][REC_F4];               // producers: (face, segment) records copied in (cp.async)
    int pws[KP_NP / 32];
    float2 uv[NT];
    float4 fpc[NWARP];
    float4 acc[TW * TH];
};

// named barriers with immediate ids (a register id makes ptxas reserve all 16 barriers of the CTA, which
// limits the CTAs per SM): 1 + b = FULL[b], 3 + b = EMPTY[b], 5 = producers only
__device__ __forceinline__ void kp_bar_sync(int id, int)
{
    if (id == 1) asm volatile("bar.sync 1, %0;" ::"n"(KP_NTH) : "memory");
    else if (id == 2) asm volatile("bar.sync 2, %0;" ::"n"(KP_NTH) : "memory");
    else if (id == 3) asm volatile("bar.sync 3, %0;" ::"n"(KP_NTH) : "memory");
    else asm volatile("bar.sync 4, %0;" ::"n"(KP_NTH) : "memory");
}
__device__ __forceinline__ void kp_bar_arrive(int id, int)
{
    if (id == 1) asm volatile("bar.arrive 1, %0;" ::"n"(KP_NTH) : "memory");
    else if (id == 2) asm volatile("bar.arrive 2, %0;" ::"n"(KP_NTH) : "memory");
    else if (id == 3) asm volatile("bar.arrive 3, %0;" ::"n"(KP_NTH) : "memory");
    else asm volatile("bar.arrive 4, %0;" ::"n"(KP_NTH) : "memory");
}
__device__ __forceinline__ void kp_pbar() { asm volatile("bar.sync 5, %0;" ::"n"(KP_NP) : "memory"); }   // producers only

// producers: stage faces j in [0, n) at the ng sub-frames taus[0..ng) into buffer b (faces: sid[j] if sid,
// else the bin entries ent[j])
__device__ __forceinline__ void kp_stage(const BinCtx &bc, const int *ent, const int *sid, int n, const float *taus,
                                         int ng, const TileCtx &tc, int W, int H, int F, TauRec *rec,
                                         uint16_t (*list)[KP_SREC], int (*cnt)[NFP], int (*cntb)[NFP], float sF, int ptid)
{
    const int npair = n * ng;
    const float inv_ng = 1.0f / (float)ng;
    for (int p = ptid; p < npair; p += KP_NP) {
        const int j = div_small(p, inv_ng), l = p - j * ng;
        const int f = sid ? sid[j] : __ldg(ent + j);
        if ((unsigned)f >= (unsigned)F) {     // never expected: bins hold valid face ids
            atomicOr(bc.status, BLUR_ST_EINTERNAL);
            continue;
        }
        const float4 *r = bc.rseg + (size_t)f * REC_F4;
        const float4 q6 = __ldg(r + 6);
        if (__float_as_int(q6.w) < 0) continue;               // skipped face (Q8, behind, bad index)
        const float tau = taus[l];
        const float D = __fmaf_rn(tau, __fmaf_rn(tau, q6.x, q6.y), q6.z);   // a1 t^2 + a2 t + a3
        if (!(fabsf(D) > EPS_D)) continue;
        const float4 b0 = __ldg(r + 7), b1 = __ldg(r + 8);
        int x0, x1, y0, y1;
        if (!tile_pixels(box_lerp(tau, b0.x, b1.x), box_lerp(tau, b0.y, b1.y), box_lerp(tau, b0.z, b1.z),
                         box_lerp(tau, b0.w, b1.w), W, H, tc, x0, x1, y0, y1))
            continue;
        FaceRec fr;
        load_rec(r, fr);
        const uint32_t fm = stage_tau<true>(fr, tau, D, x0, x1, y0, y1, tc, rec[l * n + j]);
        const uint16_t off = (uint16_t)((l * n + j) * (int)sizeof(TauRec));
        const bool back = D * sF < 0.f;   // turned away from the camera (sF: mesh orientation, 0 = unknown)
        for (uint32_t m = fm; m; m &= m - 1) {
            const int w = __ffs(m) - 1;
            if (!back) list[w][l * n + atomicAdd(&cnt[l][w], 1)] = off;
            else list[w][l * n + n - 1 - atomicAdd(&cntb[l][w], 1)] = off;
        }
    }
}

__device__ __forceinline__ void kp_cp16(void *sdst, const void *gsrc)
{
    const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gsrc) : "memory");
}

// producers: stage bin faces j in [0, n) (face ids fid[j] in shared memory) at the ng sub-frames taus[0..ng).
// The faces' records are copied into shared memory KP_NP at a time with cp.async (one L2 round trip per
// KP_NP faces, no registers held while in flight), then the (face, sub-frame) pairs are evaluated from there.
__device__ __forceinline__ void kp_stage_raw(const BinCtx &bc, const int *fid, int n, const float *taus, int ng,
                                             const TileCtx &tc, int W, int H, int F, TauRec *rec,
                                             uint16_t (*list)[KP_SREC], int (*cnt)[NFP], int (*cntb)[NFP], float sF,
                                             float4 (*raw)[REC_F4], int ptid)
{
    const float inv_ng = 1.0f / (float)ng;
    for (int fb = 0; fb < n; fb += KP_NP) {
        const int nf = min(KP_NP, n - fb);
        if (ptid < nf) {
            const int f = fid[fb + ptid];
            if ((unsigned)f < (unsigned)F) {
                const float4 *r = bc.rseg + (size_t)f * REC_F4;
#pragma unroll
                for (int i = 0; i < REC_F4; ++i) kp_cp16(&raw[ptid][i], r + i);
            } else {   // never expected: bins hold valid face ids
                atomicOr(bc.status, BLUR_ST_EINTERNAL);
                raw[ptid][6] = make_float4(0.f, 0.f, 0.f, __int_as_float(-1));
            }
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        kp_pbar();
        const int npair = nf * ng;
        for (int p = ptid; p < npair; p += KP_NP) {
            const int jj = div_small(p, inv_ng), l = p - jj * ng, j = fb + jj;
            const float4 *rr = raw[jj];
            const float4 q6 = rr[6];
            if (__float_as_int(q6.w) < 0) continue;               // skipped face (Q8, behind, bad index)
            const float tau = taus[l];
            const float D = __fmaf_rn(tau, __fmaf_rn(tau, q6.x, q6.y), q6.z);   // a1 t^2 + a2 t + a3
            if (!(fabsf(D) > EPS_D)) continue;
            const float4 b0 = rr[7], b1 = rr[8];
            int x0, x1, y0, y1;
            if (!tile_pixels(box_lerp(tau, b0.x, b1.x), box_lerp(tau, b0.y, b1.y), box_lerp(tau, b0.z, b1.z),
                             box_lerp(tau, b0.w, b1.w), W, H, tc, x0, x1, y0, y1))
                continue;
            FaceRec fr;
#pragma unroll
            for (int i = 0; i < REC_F4; ++i) fr.q[i] = rr[i];
            const uint32_t fm = stage_tau<true>(fr, tau, D, x0, x1, y0, y1, tc, rec[l * n + j]);
            const uint16_t off = (uint16_t)((l * n + j) * (int)sizeof(TauRec));
            const bool back = D * sF < 0.f;   // turned away from the camera (sF: mesh orientation, 0 = unknown)
            for (uint32_t m = fm; m; m &= m - 1) {
                const int w = __ffs(m) - 1;
                if (!back) list[w][l * n + atomicAdd(&cnt[l][w], 1)] = off;
                else list[w][l * n + n - 1 - atomicAdd(&cntb[l][w], 1)] = off;
            }
        }
        kp_pbar();   // raw is reused by the next KP_NP faces
    }
}

// producers: the next batch of an overflowed bin -- faces whose per-tau box overlaps the tile, in index order
// from fpos on (k4_raster_fwd's fallback_fill with the producer warps); returns the batch size (0: done)
__device__ __forceinline__ int kp_fill(const float4 *__restrict__ rseg, int F, float tau, const TileCtx &tc, int W, int H,
                                       int &fpos, int *sid, int *pws, int ptid)
{
    const int lane = ptid & 31, pw = ptid >> 5;
    int nb = 0;
    kp_pbar();   // the previous batch's sid has been staged by every producer
    while (fpos < F) {
        const int f = fpos + ptid;
        bool hit = false;
        if (f < F) {
            const float4 *r = rseg + (size_t)f * REC_F4;
            const float4 q6 = __ldg(r + 6);
            if (__float_as_int(q6.w) >= 0) {
                const float4 b0 = __ldg(r + 7), b1 = __ldg(r + 8);
                int x0, x1, y0, y1;
                hit = tile_pixels(box_lerp(tau, b0.x, b1.x), box_lerp(tau, b0.y, b1.y), box_lerp(tau, b0.z, b1.z),
                                  box_lerp(tau, b0.w, b1.w), W, H, tc, x0, x1, y0, y1);
            }
        }
        const unsigned m = __ballot_sync(0xffffffffu, hit);
        if (lane == 0) pws[pw] = __popc(m);
        kp_pbar();
        int pre = 0, tot = 0;
#pragma unroll
        for (int w = 0; w < KP_NP / 32; ++w) {
            const int c = pws[w];
            pre += w < pw ? c : 0;
            tot += c;
        }
        kp_pbar();
        if (nb + tot > KP_SREC) break;                   // uniform: batch full
        if (hit) sid[nb + pre + __popc(m & ((1u << lane) - 1u))] = f;
        nb += tot;
        fpos += KP_NP;
    }
    kp_pbar();   // sid[] complete before the batch is staged
    return nb;
}

// consumers: the footprint tests of one list (records of buffer rbase) against this lane's pixel
__device__ __forceinline__ void kp_vis(const unsigned char *rbase, const uint16_t *lst, int cn, int cbk, int n,
                                       float ul, float vl, float4 fc, float &zbest, int &eoff, float &tief)
{
    for (int i = 0; i < cn; ++i) {   // faces turned towards the camera
        const int off = lst[i];
        const float4 *rp = reinterpret_cast<const float4 *>(rbase + off);
        const float4 q0 = rp[0], q1 = rp[1], q2 = rp[2];
        const float e0 = edge_eval(q0.x, q0.w, q1.z, ul, vl);
        const float e1 = edge_eval(q0.y, q1.x, q1.w, ul, vl);
        const float e2 = edge_eval(q0.z, q1.y, q2.x, ul, vl);
        const float z = __fmaf_rn(q2.y, ul, __fmaf_rn(q2.z, vl, q2.w));
        const float emin = fminf(fminf(e0, e1), e2);
        tief = (emin >= 0.f && z == zbest) ? 1.f : tief;
        if (emin >= 0.f && z < zbest) { zbest = z; eoff = off; }
    }
    if (cbk) {   // the others: skipped where they are behind every pixel's winner
        float zmax = zbest;
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) zmax = fmaxf(zmax, __shfl_xor_sync(0xffffffffu, zmax, d));
        // zmax = +inf unless every pixel of the footprint has a winner.  The depth plane fma(az, ul, fma(bz, vl,
        // cz)) is monotone in ul and vl, so its minimum over the footprint's pixel centres is its value at one
        // corner: above zmax, the face cannot win or tie anywhere in the footprint.
        for (int i = n - cbk; i < n; ++i) {
            const int off = lst[i];
            const float4 *rp = reinterpret_cast<const float4 *>(rbase + off);
            const float4 q2 = rp[2];
            const float zmin = __fmaf_rn(q2.y, q2.y > 0.f ? fc.x : fc.y, __fmaf_rn(q2.z, q2.z > 0.f ? fc.z : fc.w, q2.w));
            if (zmin > zmax) continue;
            const float4 q0 = rp[0], q1 = rp[1];
            const float e0 = edge_eval(q0.x, q0.w, q1.z, ul, vl);
            const float e1 = edge_eval(q0.y, q1.x, q1.w, ul, vl);
            const float e2 = edge_eval(q0.z, q1.y, q2.x, ul, vl);
            const float z = __fmaf_rn(q2.y, ul, __fmaf_rn(q2.z, vl, q2.w));
            const float emin = fminf(fminf(e0, e1), e2);
            tief = (emin >= 0.f && z == zbest) ? 1.f : tief;
            if (emin >= 0.f && z < zbest) { zbest = z; eoff = off; }
        }
    }
}

// consumers: the lexicographic (depth, face index) z-test over both lists (exact ties, Q7; batches)
__device__ __forceinline__ void kp_vis_tie(const unsigned char *rbase, const uint16_t *lst, int cn, int cbk, int n,
                                           float ul, float vl, float &zbest, int &eoff, int &fbest)
{
    for (int ii = 0; ii < cn + cbk; ++ii) {
        const int off = lst[ii < cn ? ii : n - cbk + (ii - cn)];
        const TauRec *rr = reinterpret_cast<const TauRec *>(rbase + off);
        const float4 *rp = reinterpret_cast<const float4 *>(rr);
        const float4 q0 = rp[0], q1 = rp[1], q2 = rp[2];
        const float e0 = edge_eval(q0.x, q0.w, q1.z, ul, vl);
        const float e1 = edge_eval(q0.y, q1.x, q1.w, ul, vl);
        const float e2 = edge_eval(q0.z, q1.y, q2.x, ul, vl);
        const float z = __fmaf_rn(q2.y, ul, __fmaf_rn(q2.z, vl, q2.w));
        if (fminf(fminf(e0, e1), e2) >= 0.f && z <= zbest) {
            const int fj = rr->fid;
            if (z < zbest || fj < fbest) { zbest = z; eoff = off; fbest = fj; }
        }
    }
}

template <bool COV>
__global__ void __launch_bounds__(KP_NTH, BR_KP_MINB) k4p_raster_fwd(Tables t, float *__restrict__ out,
                                                                    int *__restrict__ ids, int ids_k)
{
    static_assert(!BR_HALF, "the pipelined forward uses the warps' 8x4 footprints");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    KpSmem &S = *reinterpret_cast<KpSmem *>(smem_raw);
    const int b = blockIdx.y, tile = blockIdx.x;
    const ImgInfo &im = t.imgs[b];
    TileCtx tc;
    tile_ctx(t, tile, tc);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 2 * GMAX_F * NFP; i += KP_NTH) { (&S.cnt[0][0][0])[i] = 0; (&S.cntb[0][0][0])[i] = 0; }
    if (threadIdx.x < NT) {
        const int lx = (warp & 1) * 8 + (lane & 7), ly = (warp >> 1) * 4 + (lane >> 3);
        S.uv[threadIdx.x] = make_float2((float)(lx - TW / 2) * tc.sx, (float)(TH / 2 - ly) * tc.sy);
        S.acc[ly * TW + lx] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (lane == 0)   // the warp footprint's corner pixel centres (the lanes' own ul, vl values)
            S.fpc[warp] = make_float4((float)((warp & 1) * 8 - TW / 2) * tc.sx, (float)((warp & 1) * 8 + 7 - TW / 2) * tc.sx,
                                      (float)(TH / 2 - (warp >> 1) * 4 - 3) * tc.sy, (float)(TH / 2 - (warp >> 1) * 4) * tc.sy);
    }
    __syncthreads();

    if (threadIdx.x >= NT) {
        // ---------------------------------------------------------------- producers
        const int ptid = threadIdx.x - NT;
        const double orient = *t.orient;
        const float sF = BR_K4P_CULL ? (orient > 0.0 ? 1.f : orient < 0.0 ? -1.f : 0.f) : 0.f;
        const bool need_empty = ids != nullptr || COV;
        const int sched_off = im.sched_off;
        int g = 0;
        for (int c = im.chunk_begin + (int)blockIdx.z; c < im.chunk_end; c += t.splits) {
            const Chunk ch = t.chunks[c];
            const size_t bi = (size_t)c * t.T + tile;
            const long long o = t.off[bi];
            const int n = (int)(t.off[bi + 1] - o);
            if (n == 0) {
                if (need_empty) {
                    const int bb = g & 1;
                    if (g >= 2) kp_bar_sync(3 + bb, KP_NTH);
                    if (ptid == 0) S.desc[bb] = KpDesc{KP_EMPTY, 0, 0, ch.k0, ch.k1, 1};
                    kp_bar_arrive(1 + bb, KP_NTH);
                    ++g;
                }
                continue;
            }
            BinCtx bc;
            bc.status = t.status;
            bc.rseg = t.rec + (size_t)(im.rec_off + (long long)ch.s * t.F) * REC_F4;
            bc.key0 = nullptr;
            bc.key1 = nullptr;
            bc.fcol = t.fcol;
            bc.ent = t.entries + o;
            bc.n = n;
            bc.fb = o + n > t.cap;
            if (!bc.fb && n <= KP_SREC) {
                const int Gs = min(GMAX_F, group_div(KP_SREC, n));
                kp_pbar();   // every producer is done with the previous chunk's face ids
                for (int j = ptid; j < n; j += KP_NP) S.sid[j] = __ldg(bc.ent + j);
                for (int kg = ch.k0; kg < ch.k1; kg += Gs) {
                    const int ng = min(Gs, ch.k1 - kg), bb = g & 1;
                    if (g >= 2) kp_bar_sync(3 + bb, KP_NTH);   // buffer bb consumed (and its counters cleared)
                    if (ptid < ng) S.taus[bb][ptid] = t.sched_tau[sched_off + kg + ptid];
                    if (ptid == 0) S.desc[bb] = KpDesc{KP_GROUP, n, ng, kg, 0, 0};
                    kp_pbar();
                    kp_stage_raw(bc, S.sid, n, S.taus[bb], ng, tc, t.W, t.H, t.F, S.rec[bb], S.list[bb], S.cnt[bb],
                                 S.cntb[bb], sF, S.raw, ptid);
                    kp_bar_arrive(1 + bb, KP_NTH);
                    ++g;
                }
            } else {
                for (int k = ch.k0; k < ch.k1; ++k) {
                    const float tau = t.sched_tau[sched_off + k];
                    int base = 0, fpos = 0;
                    while (true) {
                        const int bb = g & 1;
                        if (g >= 2) kp_bar_sync(3 + bb, KP_NTH);
                        int nb;
                        if (bc.fb) nb = kp_fill(bc.rseg, t.F, tau, tc, t.W, t.H, fpos, S.sid, S.pws, ptid);
                        else nb = min(KP_SREC, n - base);
                        const bool last = nb == 0 || (!bc.fb && base + nb >= n);
                        if (ptid == 0) { S.taus[bb][0] = tau; S.desc[bb] = KpDesc{KP_BATCH, nb, 1, k, base, last ? 1 : 0}; }
                        kp_pbar();
                        if (nb > 0)
                            kp_stage(bc, bc.ent + base, bc.fb ? S.sid : nullptr, nb, S.taus[bb], 1, tc, t.W, t.H, t.F, S.rec[bb],
                                     S.list[bb], S.cnt[bb], S.cntb[bb], sF, ptid);
                        kp_bar_arrive(1 + bb, KP_NTH);
                        ++g;
                        base += nb;
                        if (last) break;
                    }
                }
            }
        }
        const int bb = g & 1;
        if (g >= 2) kp_bar_sync(3 + bb, KP_NTH);
        if (ptid == 0) S.desc[bb] = KpDesc{KP_END, 0, 0, 0, 0, 0};
        kp_bar_arrive(1 + bb, KP_NTH);
        return;
    }

    // -------------------------------------------------------------------- consumers (8 warps, one footprint each)
    const int lx = (warp & 1) * 8 + (lane & 7), ly = (warp >> 1) * 4 + (lane >> 3);
    const int px = tc.px0 + lx, py = tc.py0 + ly;
    const bool inimg = px < t.W && py < t.H;
    const int myp = ly * TW + lx;
    // per-sub-frame batch state (long and overflowed bins)
    float bz = __int_as_float(0x7f800000), pr = 0.f, pg = 0.f, pb = 0.f;
    int bfb = 0x7fffffff, bfid = -1;
    bool has = false;
    for (int g = 0;; ++g) {
        const int bb = g & 1;
        kp_bar_sync(1 + bb, KP_NTH);
        const KpDesc d = S.desc[bb];
        if (d.kind == KP_END) break;
        const unsigned char *rbase = reinterpret_cast<const unsigned char *>(S.rec[bb]);
        const float2 uvp = S.uv[threadIdx.x];
        const float ul = uvp.x, vl = uvp.y;
        if (d.kind == KP_EMPTY) {
            if (ids && inimg && ids_k >= d.kg && ids_k < d.k1) ids[((size_t)b * t.H + py) * t.W + px] = -1;
            if (COV) {
                const unsigned m = __ballot_sync(0xffffffffu, !inimg);
                if (lane == 0)
                    for (int k = d.kg; k < d.k1; ++k) t.covbits[cov_word(t, im, k, tile) + warp] = m;
            }
        } else if (d.kind == KP_GROUP) {
            const int n = d.n;
            uint16_t *vrow = (n <= VIS_MAXN && t.vis) ? t.vis + ((size_t)(im.cov_off + d.kg) * t.T + tile) * (TW * TH) + myp : nullptr;
            const uint16_t *lst = S.list[bb][warp];
            const float4 fc = S.fpc[warp];
            for (int l = 0; l < d.ng; ++l, lst += n) {
                const int cn = S.cnt[bb][l][warp], cbk = S.cntb[bb][l][warp];
                float zbest = __int_as_float(0x7f800000), tief = 0.f;
                int eoff = -1;
                kp_vis(rbase, lst, cn, cbk, n, ul, vl, fc, zbest, eoff, tief);
                if (__any_sync(0xffffffffu, tief != 0.f)) {   // exact depth tie in the warp: face indices decide (Q7)
                    zbest = __int_as_float(0x7f800000);
                    eoff = -1;
                    int fbest = 0x7fffffff;
                    kp_vis_tie(rbase, lst, cn, cbk, n, ul, vl, zbest, eoff, fbest);
                }
                __syncwarp();
                if (lane == 0) { S.cnt[bb][l][warp] = 0; S.cntb[bb][l][warp] = 0; }
                const int ebest = eoff >= 0 ? eoff / (int)sizeof(TauRec) - l * n : -1;
                int fid = -1;
                if (ebest >= 0) {
                    const TauRec &rw = *reinterpret_cast<const TauRec *>(rbase + eoff);
                    float r_, g_, b_;
                    shade(rw, t.fcol, ul, vl, r_, g_, b_);      // Eq.9
                    float4 a = S.acc[myp];
                    a.x += r_; a.y += g_; a.z += b_; a.w += 1.f;
                    S.acc[myp] = a;
                    fid = rw.fid;
                }
                if (ids && inimg && d.kg + l == ids_k) ids[((size_t)b * t.H + py) * t.W + px] = fid;
                if (vrow) {   // visibility cache for K6
                    *vrow = ebest >= 0 ? (uint16_t)ebest : (uint16_t)0xFFFF;
                    vrow += (size_t)t.T * (TW * TH);
                }
                if (COV) {   // soft path: which pixels of the warp are covered at this sub-frame
                    const unsigned m = __ballot_sync(0xffffffffu, ebest >= 0 || !inimg);
                    if (lane == 0) t.covbits[cov_word(t, im, d.kg + l, tile) + warp] = m;
                }
            }
        } else {   // KP_BATCH: one sub-frame d.kg, records of bin slots [d.k1, d.k1 + n); d.last ends it
            const int n = d.n;
            if (n > 0) {
                const uint16_t *lst = S.list[bb][warp];
                const int cn = S.cnt[bb][0][warp], cbk = S.cntb[bb][0][warp];
                int eoff = -1;
                kp_vis_tie(rbase, lst, cn, cbk, n, ul, vl, bz, eoff, bfb);
                __syncwarp();
                if (lane == 0) { S.cnt[bb][0][warp] = 0; S.cntb[bb][0][warp] = 0; }
                if (eoff >= 0) {   // winner changed in this batch: shade now (Eq.9)
                    const TauRec &rw = *reinterpret_cast<const TauRec *>(rbase + eoff);
                    shade(rw, t.fcol, ul, vl, pr, pg, pb);
                    has = true;
                    bfid = rw.fid;
                }
            }
            if (d.last) {
                if (has) {
                    float4 a = S.acc[myp];
                    a.x += pr; a.y += pg; a.z += pb; a.w += 1.f;
                    S.acc[myp] = a;
                }
                if (ids && inimg && d.kg == ids_k) ids[((size_t)b * t.H + py) * t.W + px] = has ? bfid : -1;
                if (COV) {
                    const unsigned m = __ballot_sync(0xffffffffu, has || !inimg);
                    if (lane == 0) t.covbits[cov_word(t, im, d.kg, tile) + warp] = m;
                }
                bz = __int_as_float(0x7f800000);
                bfb = 0x7fffffff;
                bfid = -1;
                has = false;
            }
        }
        kp_bar_arrive(3 + bb, KP_NTH);
    }
    if (inimg && out) {   // out == null: coverage-only pass (soft backward without a preceding forward)
        const float inv = 1.0f / (float)im.N;
        const float4 a = S.acc[myp];
        const float4 v = make_float4(a.x * inv, a.y * inv, a.z * inv, a.w * inv);
        const size_t pix = ((size_t)b * t.H + py) * t.W + px;
        if (t.splits == 1) reinterpret_cast<float4 *>(out)[pix] = v;
        else t.part[(size_t)blockIdx.z * ((size_t)t.B * t.H * t.W) + pix] = v;
    }
}

template <bool COV>
static cudaError_t launch_fwd_pipe(const Tables &t, float *out, int *ids, int ids_k, cudaStream_t st)
{
    dim3 grid(t.T, t.B, t.splits);
    const int smem = (int)sizeof(KpSmem);
    cudaError_t e = cudaFuncSetAttribute(k4p_raster_fwd<COV>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    k4p_raster_fwd<COV><<<grid, KP_NTH, smem, st>>>(t, out, ids, ids_k);
    return cudaGetLastError();
}

// BLURRAST_FWD=pipe: the warp-specialised k4p_raster_fwd instead of k4l_raster_fwd (A/B; measured slower,
// DESIGN.md section 4)
static bool pipe_fwd_on()
{
    const char *s = std::getenv("BLURRAST_FWD");
    return s && std::strcmp(s, "pipe") == 0;
}

// BLURRAST_LEAN_FWD=0: the fast solver's timed forward takes k4_raster_fwd instead (A/B)
static bool lean_fwd_off()
{
    const char *s = std::getenv("BLURRAST_LEAN_FWD");
    return s && s[0] == '0';
}

// ------------------------------------------------------------------ backward
//
// Visibility as in the forward pass.  Then, per (tile, sub-frame): the face's gradient is linear in
// g = dL/dI_k and w_i(p) is affine in the tile-local pixel position, so each face only needs nine
// moments of g over the pixels it won: m0 = sum g, mu = sum u g, mv = sum v g.  Then (Eq.9 and
// dw/dv_i = -w_i dw/dp)
//   dL/dc_i = (A_i mu + B_i mv + G_i m0) / |D|
//   dL/dv_i = -( A_i (PA.mu) + B_i (PA.mv) + G_i (PA.m0),  same with PB ) / D^2,
//   PA = sum_j A_j c_j, PB = sum_j B_j c_j  (A, B, G the sign-normalised numerator coefficients).
// The moments are reduced pixel-parallel: the won pixels are counting-sorted by winning slot
// (integer shared-memory atomics), every thread forms the 9 moment terms of one won pixel, a warp
// segmented scan sums runs of equal slots, and each face thread combines its partial sums and
// evaluates the closed form.  Face gradients accumulate in registers over the chunk's sub-frames
// (slot == thread) and are flushed with one vector RED per (vertex, keyframe) at the chunk's end.

// Record of a (face, segment) coefficient record at tau for this tile, written unconditionally (the
// cached-visibility backward stages only faces that won a pixel in the forward, whose records the
// forward built with the same arithmetic).
__device__ __forceinline__ void stage_rec(const FaceRec &fr, float tau, const TileCtx &tc, TauRec &out)
{
    const float4 q6 = fr.q[6];
    const float D = __fmaf_rn(tau, __fmaf_rn(tau, q6.x, q6.y), q6.z);
    const float sg = D < 0.f ? -1.f : 1.f;
    const float invD = 1.0f / fabsf(D);
    float A[3], B[3], G[3];
    const float *ef = reinterpret_cast<const float *>(fr.q);
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        float al, be, gp;
        rec_edge_at(fr.q[2 * i], fr.q[2 * i + 1], tau, tc.uc, tc.vc, al, be, gp);
        A[i] = al * sg;
        B[i] = be * sg;
        G[i] = gp * sg;
    }
    out.a[0] = A[0]; out.a[1] = A[1]; out.a[2] = A[2];
    out.b[0] = B[0]; out.b[1] = B[1]; out.b[2] = B[2];
    out.g[0] = G[0]; out.g[1] = G[1]; out.g[2] = G[2];
    out.az = 0.f;       // depth plane unused by the gather
    out.bz = 0.f;
    out.cz = 0.f;
    out.invD = invD;
    out.fid = __float_as_int(q6.w);
}

// stage the won (face, sub-frame) pairs of bin slots [0, n) at the ng sub-frames: rec[l * n + j]
// (won[l * n + j] == stamp marks them: no clearing between groups)
__device__ __forceinline__ void stage_won(const BinCtx &bc, int n, const float *taus, int ng, const TileCtx &tc, int F,
                                          const unsigned int *won, unsigned int stamp, TauRec *rec)
{
    const float inv_ng = 1.0f / (float)ng;
    for (int p = threadIdx.x; p < n * ng; p += NT) {
        const int j = div_small(p, inv_ng), l = p - j * ng;
        if (won[l * n + j] != stamp) continue;
        const int f = __ldg(bc.ent + j);
        if ((unsigned)f >= (unsigned)F) {
            atomicOr(bc.status, BLUR_ST_EINTERNAL);
            continue;
        }
        FaceRec fr;
        load_rec(bc.rseg + (size_t)f * REC_F4, fr);
        stage_rec(fr, taus[l], tc, rec[l * n + j]);
    }
}

template <int MODE>
struct BwdSmem {
    TauRec rec[SREC_B];
    float4 vtx[MODE == 2 ? 3 * SREC_B : 1];
    uint32_t wm[NFP * (SREC_B / 32 + GMAX_B)];
    int sid[SREC_B];
    short win[GMAX_B][TW * TH];   // winning slot per (sub-frame of the group, pixel), -1 none
    int cnt[SREC_B];          // won-pixel count per staged slot (key)
    int off[SREC_B];          // exclusive prefix of cnt
    int key[TW * TH];         // sorted won pixels: slot
    int pix[TW * TH];         //                    pixel
    float mom[9][TW * TH];    // segment partial moments at the run's last position (per warp)
    float4 g[TW * TH];        // dL/dI / N of the tile
    float taus[GMAX_B];
    int wsum[NWARP];
    unsigned int won[SREC_B];   // cached visibility: group stamp of the (sub-frame, slot) pairs that won a pixel
    int pxinfo[NT];                  // the thread's pixel: myp | in-image << 8 (reloaded rather than re-derived)
};

// block-wide exclusive scan of cnt[0..nb) (nb <= 2 NT) into off[]; returns the total
template <class Sm>
__device__ __forceinline__ int scan_counts(Sm &S, int nb)
{
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int j0 = 2 * tid;
    const int c0 = j0 < nb ? S.cnt[j0] : 0, c1 = j0 + 1 < nb ? S.cnt[j0 + 1] : 0;
    int x = c0 + c1;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) S.wsum[warp] = x;
    __syncthreads();
    int pre = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < NWARP; ++w) {
        const int v = S.wsum[w];
        pre += w < warp ? v : 0;
        tot += v;
    }
    const int ex = pre + x - (c0 + c1);
    if (j0 < nb) S.off[j0] = ex;
    if (j0 + 1 < nb) S.off[j0 + 1] = ex + c0;
    return tot;
}


// Reduce the moments of the won pixels whose winner lies in the staged batch [base, base+nb)
// (records rec[0..nb)) and give each face with winners its closed-form gradient: persistent slots
// (slot == thread) accumulate in registers across the chunk, the others flush immediately.
template <class Sm>
__device__ __forceinline__ void bwd_gather(Sm &S, const TauRec *rec, const Tables &t, const ImgInfo &im, int s,
                                           float tau, int base, int nb, bool persist_ok, int ebest, int myp,
                                           const TileCtx &tc, FaceAcc &acc, float *dC)
{
    const int tid = threadIdx.x, lane = tid & 31;
    // S.cnt[0..nb) is zero on entry (cleared at kernel start and by the previous gather's combine)
    const int e = ebest - base;
    const bool mine = ebest >= 0 && e >= 0 && e < nb;
    int rank = 0;
    if (mine) rank = atomicAdd(&S.cnt[e], 1);
    __syncthreads();
    if ((tid >> 5) == 0) {   // one warp scans the <= SREC_B counts (no block barrier inside)
        const int per = (nb + 31) >> 5, j0 = lane * per, j1 = min(nb, j0 + per);
        int sum = 0;
        for (int j = j0; j < j1; ++j) sum += S.cnt[j];
        int x = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        int run = x - sum;
        for (int j = j0; j < j1; ++j) { S.off[j] = run; run += S.cnt[j]; }
        if (lane == 31) S.wsum[0] = x;
    }
    __syncthreads();
    const int total = S.wsum[0];
    if (mine) {
        const int pos = S.off[e] + rank;
        S.key[pos] = e;
        S.pix[pos] = myp;
    }
    __syncthreads();
    // moment terms of one won pixel per thread, warp segmented inclusive scan over equal slots
    {
        int key = -1 - tid;   // unique keys for idle threads (never merged)
        float m[9];
#pragma unroll
        for (int q = 0; q < 9; ++q) m[q] = 0.f;
        if (tid < total) {
            key = S.key[tid];
            const int p = S.pix[tid];
            const float4 g = S.g[p];
            const float ul = (float)((p & (TW - 1)) - TW / 2) * tc.sx;
            const float vl = (float)(TH / 2 - (p / TW)) * tc.sy;
            m[0] = g.x; m[1] = g.y; m[2] = g.z;
            m[3] = ul * g.x; m[4] = ul * g.y; m[5] = ul * g.z;
            m[6] = vl * g.x; m[7] = vl * g.y; m[8] = vl * g.z;
        }
        // run heads (a lane whose key differs from the previous lane's) once, then each step adds the
        // value d lanes up iff that lane is still in this lane's run: lane - d >= run start
        const int kprev = __shfl_up_sync(0xffffffffu, key, 1);
        const unsigned heads = __ballot_sync(0xffffffffu, lane == 0 || kprev != key);
        const int run = lane - (31 - __clz(heads & (0xffffffffu >> (31 - lane))));   // lanes before this one in the run
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const bool take = run >= d;
#pragma unroll
            for (int q = 0; q < 9; ++q) {
                const float v = __shfl_up_sync(0xffffffffu, m[q], d);
                if (take) m[q] += v;
            }
        }
        const int knext = __shfl_down_sync(0xffffffffu, key, 1);
        if (tid < total && (lane == 31 || tid == total - 1 || knext != key)) {
#pragma unroll
            for (int q = 0; q < 9; ++q) S.mom[q][tid] = m[q];
        }
    }
    __syncthreads();
    for (int j = tid; j < nb; j += NT) {
        const int c = S.cnt[j];
        if (c == 0) continue;
        S.cnt[j] = 0;                                  // ready for the next gather (see entry)
        const int st = S.off[j], en = st + c - 1;
        float m[9];
#pragma unroll
        for (int q = 0; q < 9; ++q) m[q] = S.mom[q][en];
        for (int i = st | 31; i < en; i += 32)        // partial sums ending at warp boundaries
#pragma unroll
            for (int q = 0; q < 9; ++q) m[q] += S.mom[q][i];
        float dv[6], dc[9];
        face_grad(rec[j], m, t.fcol, dv, dc);
        if (persist_ok && j == tid) {
#pragma unroll
            for (int i = 0; i < 6; ++i) {
                acc.k0[i] = __fmaf_rn(1.f - tau, dv[i], acc.k0[i]);
                acc.k1[i] = __fmaf_rn(tau, dv[i], acc.k1[i]);
            }
#pragma unroll
            for (int i = 0; i < 9; ++i) acc.c[i] += dc[i];
        } else {
            float a0[6], a1[6];
#pragma unroll
            for (int i = 0; i < 6; ++i) { a0[i] = (1.f - tau) * dv[i]; a1[i] = tau * dv[i]; }
            flush(t, im, s, rec[j].fid, a0, a1, dc, dC);
        }
    }
    __syncthreads();
}

template <int MODE>
__global__ void __launch_bounds__(NT, BR_K6_MINB) k6_raster_bwd(Tables t, const float *__restrict__ grad, float *__restrict__ dC)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    BwdSmem<MODE> &S = *reinterpret_cast<BwdSmem<MODE> *>(smem_raw);
    const int b = blockIdx.y, tile = blockIdx.x;
    const ImgInfo &im = t.imgs[b];
    const int N = im.N, c_begin = im.chunk_begin, c_end = im.chunk_end, sched_off = im.sched_off;
    const long long rec_off = im.rec_off;
    TileCtx tc;
    tile_ctx(t, tile, tc);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int lx = (warp & 1) * 8 + (lane & 7), ly = (warp >> 1) * 4 + (lane >> 3);
    const int px = tc.px0 + lx, py = tc.py0 + ly;
    const bool inimg = px < t.W && py < t.H;
    const float ul = (float)(lx - TW / 2) * tc.sx;
    const float vl = (float)(TH / 2 - ly) * tc.sy;
    const int myp = ly * TW + lx;
    {
        float4 g = make_float4(0.f, 0.f, 0.f, 0.f);
        if (inimg) {
            g = __ldg(reinterpret_cast<const float4 *>(grad) + ((size_t)b * t.H + py) * t.W + px);
            const float inv = 1.0f / (float)N;   // dI/dI_k = 1/N (uniform mean)
            g.x *= inv; g.y *= inv; g.z *= inv; g.w = 0.f;
        }
        S.g[myp] = g;
    }
    for (int j = threadIdx.x; j < SREC_B; j += NT) S.cnt[j] = 0;   // invariant of bwd_gather
    S.pxinfo[threadIdx.x] = myp | (inimg ? 0x100 : 0);
    for (int j = threadIdx.x; j < SREC_B; j += NT) S.won[j] = 0xFFFFFFFFu;
    unsigned int stamp = 0;   // group counter of the cached path (won flags)
    __syncthreads();
    unsigned long long d0 = 0, d1 = 0, d2 = 0;

    for (int c = c_begin + (int)blockIdx.z; c < c_end; c += t.splits) {
        const Chunk ch = t.chunks[c];
        const size_t bi = (size_t)c * t.T + tile;
        const long long o = t.off[bi];
        const int n = (int)(t.off[bi + 1] - o);
        if (n == 0) continue;
        BinCtx bc;
        bc.status = t.status;
        bc.rseg = t.rec + (size_t)(rec_off + (long long)ch.s * t.F) * REC_F4;
        bc.key0 = t.key + im.key_off + (size_t)ch.s * t.V;
        bc.key1 = bc.key0 + t.V;
        bc.fcol = t.fcol;
        bc.ent = t.entries + o;
        bc.n = n;
        bc.fb = o + n > t.cap;
        FaceAcc acc;
        acc_zero(acc);
        if (MODE == 0 && t.vis && !bc.fb && n <= VIS_MAXN) {
            if (t.vis_gathered) continue;   // taken by k6v_raster_bwd (k_gather.cu)
            // visibility from the forward's buffer: stage only the (face, sub-frame) pairs that won
            const int Gs = min(GMAX_B, group_div(SREC_B, n));
            for (int kg = ch.k0; kg < ch.k1; kg += Gs) {
                const int ng = min(Gs, ch.k1 - kg);
                ++stamp;
                if (threadIdx.x < ng) S.taus[threadIdx.x] = t.sched_tau[sched_off + kg + threadIdx.x];
                __syncthreads();
                const int pi = S.pxinfo[threadIdx.x], mp = pi & 0xFF;
                const uint16_t *vrow = t.vis + ((size_t)(im.cov_off + kg) * t.T + tile) * (TW * TH) + mp;
                for (int l = 0; l < ng; ++l, vrow += (size_t)t.T * (TW * TH)) {
                    const uint16_t v = *vrow;
                    const int e = ((pi & 0x100) && v != 0xFFFF) ? (int)v : -1;
                    S.win[l][mp] = (short)e;
                    if (e >= 0) S.won[l * n + e] = stamp;
                }
                __syncthreads();
                stage_won(bc, n, S.taus, ng, tc, t.F, S.won, stamp, S.rec);
                __syncthreads();
                for (int l = 0; l < ng; ++l) {
                    const int mq = S.pxinfo[threadIdx.x] & 0xFF;
                    bwd_gather(S, S.rec + l * n, t, im, ch.s, S.taus[l], 0, n, true, S.win[l][mq], mq, tc, acc, dC);
                }
            }
        } else if (!bc.fb && n <= SREC_B) {
            const int Gs = min(GMAX_B, group_div(SREC_B, n)), nw = (n + 31) >> 5;
            for (int kg = ch.k0; kg < ch.k1; kg += Gs) {
                const int ng = min(Gs, ch.k1 - kg);
                clear_words(S.wm, ng * NFP * nw);
                if (threadIdx.x < ng) S.taus[threadIdx.x] = t.sched_tau[sched_off + kg + threadIdx.x];
                __syncthreads();
                stage_group<false, MODE>(bc, n, 0, S.taus, ng, tc, t.W, t.H, t.F, S.sid, S.rec, S.vtx, S.wm, d2);
                __syncthreads();
                for (int l = 0; l < ng; ++l) {       // visibility for the group (no barriers)
                    float zbest = __int_as_float(0x7f800000);
                    int ebest = -1, fbest = 0x7fffffff;
                    const uint32_t *wml = S.wm + (l * NFP + fp_of(warp, lane)) * nw;
                    bool tie = true;
                    if (MODE != 2) tie = vis_mask_fast<false, MODE>(S.rec + l * n, wml, nw, ul, vl, zbest, ebest, d0, d1, false);
                    if (__any_sync(0xffffffffu, tie)) {
                        zbest = __int_as_float(0x7f800000);
                        ebest = -1;
                        vis_mask<false, MODE>(S.rec + l * n, S.vtx + 3 * l * n, wml, nw, 0, ul, vl, zbest, ebest, fbest,
                                              d0, d1, false);
                    }
                    S.win[l][myp] = (short)(inimg ? ebest : -1);
                }
                __syncthreads();
                for (int l = 0; l < ng; ++l)
                    bwd_gather(S, S.rec + l * n, t, im, ch.s, S.taus[l], 0, n, true, S.win[l][myp], myp, tc, acc, dC);
            }
        } else {
            for (int k = ch.k0; k < ch.k1; ++k) {
                const float tau = t.sched_tau[sched_off + k];
                float zbest = __int_as_float(0x7f800000);
                int ebest = -1, fbest = 0x7fffffff;
                int base = 0, fpos = 0;
                if (threadIdx.x == 0) S.taus[0] = tau;
                while (true) {                         // visibility over all batches
                    const int nb = next_batch(bc, t.F, tau, tc, t.W, t.H, SREC_B, base, fpos, S.sid, S.wsum);
                    if (nb == 0) break;
                    const int nw = (nb + 31) >> 5;
                    clear_words(S.wm, NFP * nw);
                    __syncthreads();
                    stage_group<false, MODE>(bc, nb, base, S.taus, 1, tc, t.W, t.H, t.F, S.sid, S.rec, S.vtx, S.wm, d2);
                    __syncthreads();
                    vis_mask<false, MODE>(S.rec, S.vtx, S.wm + fp_of(warp, lane) * nw, nw, base, ul, vl, zbest, ebest, fbest, d0, d1,
                                          false);
                    if (ebest >= base) fbest = S.rec[ebest - base].fid;
                    base += nb;
                    __syncthreads();
                }
                if (!inimg) ebest = -1;
                base = 0;
                fpos = 0;
                while (true) {                         // re-stage each batch and gather
                    const int nb = next_batch(bc, t.F, tau, tc, t.W, t.H, SREC_B, base, fpos, S.sid, S.wsum);
                    if (nb == 0) break;
                    const int nw = (nb + 31) >> 5;
                    clear_words(S.wm, NFP * nw);
                    __syncthreads();
                    stage_group<false, MODE>(bc, nb, base, S.taus, 1, tc, t.W, t.H, t.F, S.sid, S.rec, S.vtx, S.wm, d2);
                    __syncthreads();
                    bwd_gather(S, S.rec, t, im, ch.s, tau, base, nb, false, ebest, myp, tc, acc, dC);
                    base += nb;
                }
            }
        }
        if (!bc.fb && n <= SREC_B && (int)threadIdx.x < n) {   // persistent slots (both grouped paths)
            bool nz = false;
#pragma unroll
            for (int i = 0; i < 9; ++i) nz |= acc.c[i] != 0.f;
#pragma unroll
            for (int i = 0; i < 6; ++i) nz |= (acc.k0[i] != 0.f) | (acc.k1[i] != 0.f);
            if (nz) flush(t, im, ch.s, __ldg(bc.ent + threadIdx.x), acc.k0, acc.k1, acc.c, dC);
        }
    }
}

// ------------------------------------------------------------------ backward without the visibility buffer
//
// k6_raster_bwd_fx recomputes the visibility with the forward's own stage + per-warp mask walk (the
// winners are never stored in HBM), and reduces the nine moments of every staged (face,
// sub-frame) record in fixed point: each pixel adds q = round(g * 2^e) and q * (x - TW/2), q * (TH/2 - y)
// (g = dL/dI / N per channel; 2^e a power of two per tile with max |q| <= 2^19, so every sum of the
// 256 pixels stays below 2^31) to its winner's slot with native 32-bit shared-memory atomics.  Integer
// sums are exact and independent of the order the pixels arrive in (deterministic); the one rounding per
// pixel is below 2^-20 of the tile's largest |g|.  The moments convert back (m0 = M0 2^-e, mu = Mu 2^-e sx,
// mv = Mv 2^-e sy) and the closed form of face_grad gives each record's gradient; the slot's thread adds
// it over the chunk's sub-frames, split (1 - tau, tau) onto the keyframes (Eq.5-6).

template <int MODE>
struct BwdFxSmem {
    TauRec rec[SREC_B];
    float4 vtx[MODE == 2 ? 3 * SREC_B : 1];
    uint32_t wm[NFP * (SREC_B / 32 + GMAX_B)];
    int sid[SREC_B];
    int imom[SREC_B][10];    // fixed-point moments M0 (rgb), Mu (rgb), Mv (rgb) and the won count per record
    int4 qg[TW * TH];        // the tile's fixed-point pixel gradients q (rgb)
    float taus[GMAX_B];
    int wsum[NWARP];
    float red[NWARP];
    unsigned int won[SREC_B];   // cached visibility: group stamp of the (sub-frame, slot) pairs that won a pixel
};

// add the pixel's fixed-point moment terms to its winning record's slot
__device__ __forceinline__ void add_moments(int *m, int4 q, int dx, int dy)
{
    atomicAdd(m + 0, q.x); atomicAdd(m + 1, q.y); atomicAdd(m + 2, q.z);
    atomicAdd(m + 3, q.x * dx); atomicAdd(m + 4, q.y * dx); atomicAdd(m + 5, q.z * dx);
    atomicAdd(m + 6, q.x * dy); atomicAdd(m + 7, q.y * dy); atomicAdd(m + 8, q.z * dy);
    atomicAdd(m + 9, 1);
}

#ifndef BR_FX_RUNS
#define BR_FX_RUNS 1   // 1: a warp's 8-pixel row runs of equal winners add their moments once (prefix differences)
#endif
// Run-aggregated form of add_moments for a whole warp (8x4 footprint, lanes 8r..8r+7 = one 8-pixel row):
// each run of equal keys (the winner's slot, -1 none) in a row adds its sums once, from the lanes' inclusive
// row prefixes P of q and q dx (built once per tile); q dy = dy x sum q (one row).  The same integers as the
// per-pixel atomics (exact, order-independent).  All 32 lanes must call it.
__device__ __forceinline__ void run_moments(int *imom, int key, int lane, const int P[6], int dy)
{
    const int c = lane & 7;
    const int kp = __shfl_up_sync(0xffffffffu, key, 1), kn = __shfl_down_sync(0xffffffffu, key, 1);
    const bool st = c == 0 || kp != key, en = c == 7 || kn != key;
    const unsigned sm = __ballot_sync(0xffffffffu, st);
    const int s = 31 - __clz(sm & (0xffffffffu >> (31 - lane)));   // first lane of this lane's run
    const int src = (s & 7) ? s - 1 : s;
    int b[6];
#pragma unroll
    for (int i = 0; i < 6; ++i) {
        b[i] = __shfl_sync(0xffffffffu, P[i], src);
        if ((s & 7) == 0) b[i] = 0;
    }
    if (en && key >= 0) {
        int *m = imom + 10 * key;
        const int m0 = P[0] - b[0], m1 = P[1] - b[1], m2 = P[2] - b[2];
        atomicAdd(m + 0, m0); atomicAdd(m + 1, m1); atomicAdd(m + 2, m2);
        atomicAdd(m + 3, P[3] - b[3]); atomicAdd(m + 4, P[4] - b[4]); atomicAdd(m + 5, P[5] - b[5]);
        atomicAdd(m + 6, m0 * dy); atomicAdd(m + 7, m1 * dy); atomicAdd(m + 8, m2 * dy);
        atomicAdd(m + 9, lane - s + 1);
    }
}

// read, clear and convert the fixed-point moments of one record (returns the won count)
__device__ __forceinline__ int take_moments(int *m, float inv, float sx, float sy, float f[9])
{
    const int cnt = m[9];
    if (cnt == 0) return 0;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        f[q] = (float)m[q] * inv;
        f[3 + q] = (float)m[3 + q] * inv * sx;
        f[6 + q] = (float)m[6 + q] * inv * sy;
    }
#pragma unroll
    for (int q = 0; q < 10; ++q) m[q] = 0;
    return cnt;
}

template <int MODE>
__device__ __forceinline__ void k6_fx_tile(const Tables &t, const float *__restrict__ grad, float *__restrict__ dC,
                                           int b, int tile, int z, BwdFxSmem<MODE> &S);

template <int MODE>
__global__ void __launch_bounds__(NT, BR_K6_MINB) k6_raster_bwd_fx(Tables t, const float *__restrict__ grad,
                                                                  float *__restrict__ dC)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    BwdFxSmem<MODE> &S = *reinterpret_cast<BwdFxSmem<MODE> *>(smem_raw);
    if (!t.vis_gathered) {   // grid: tiles x images x splits
        k6_fx_tile<MODE>(t, grad, dC, blockIdx.y, blockIdx.x, blockIdx.z, S);
        return;
    }
    // after k6v_raster_bwd (k_gather.cu): only the (image, tile)s it listed as having chunks left, grid-stride
    const int nl = *t.vg_count;
    for (int i = blockIdx.x; i < nl; i += gridDim.x) {
        const int item = t.vg_list[i];
        __syncthreads();   // the previous item's shared memory is no longer read
        k6_fx_tile<MODE>(t, grad, dC, item / t.T, item % t.T, blockIdx.z, S);
    }
}

template <int MODE>
__device__ __forceinline__ void k6_fx_tile(const Tables &t, const float *__restrict__ grad, float *__restrict__ dC,
                                           int b, int tile, int z, BwdFxSmem<MODE> &S)
{
    const ImgInfo &im = t.imgs[b];
    const int N = im.N, c_begin = im.chunk_begin, c_end = im.chunk_end, sched_off = im.sched_off;
    const long long rec_off = im.rec_off;
    TileCtx tc;
    tile_ctx(t, tile, tc);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int lx = (warp & 1) * 8 + (lane & 7), ly = (warp >> 1) * 4 + (lane >> 3);
    const int px = tc.px0 + lx, py = tc.py0 + ly;
    const bool inimg = px < t.W && py < t.H;
    const float ul = (float)(lx - TW / 2) * tc.sx;
    const float vl = (float)(TH / 2 - ly) * tc.sy;
    const int myp = ly * TW + lx;
    // the tile's pixel gradients in fixed point: scale 2^e with max |g| 2^e < 2^19
    float4 g = make_float4(0.f, 0.f, 0.f, 0.f);
    if (inimg) {
        g = __ldg(reinterpret_cast<const float4 *>(grad) + ((size_t)b * t.H + py) * t.W + px);
        const float inv = 1.0f / (float)N;   // dI/dI_k = 1/N (uniform mean)
        g.x *= inv; g.y *= inv; g.z *= inv;
    }
    float gm = fmaxf(fmaxf(fabsf(g.x), fabsf(g.y)), fabsf(g.z));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) gm = fmaxf(gm, __shfl_xor_sync(0xffffffffu, gm, o));
    if (lane == 0) S.red[warp] = gm;
    for (int j = threadIdx.x; j < SREC_B * 10; j += NT) (&S.imom[0][0])[j] = 0;
    __syncthreads();
    gm = 0.f;
#pragma unroll
    for (int w = 0; w < NWARP; ++w) gm = fmaxf(gm, S.red[w]);
    int ex = 0;
    if (gm > 0.f) frexpf(gm, &ex);                 // gm = m 2^ex, m in [0.5, 1)
    ex = min(max(ex, -100), 100);
    const float scale = ldexpf(1.0f, 19 - ex), inv_scale = ldexpf(1.0f, ex - 19);
    S.qg[myp] = make_int4(__float2int_rn(g.x * scale), __float2int_rn(g.y * scale), __float2int_rn(g.z * scale), 0);
    const int dx = lx - TW / 2, dy = TH / 2 - ly;
#if BR_FX_RUNS
    int P[6];   // inclusive prefixes over this lane's 8-pixel row segment of q and q dx (run_moments)
    {
        const int4 q0 = S.qg[myp];
        P[0] = q0.x; P[1] = q0.y; P[2] = q0.z; P[3] = q0.x * dx; P[4] = q0.y * dx; P[5] = q0.z * dx;
#pragma unroll
        for (int d = 1; d < 8; d <<= 1)
#pragma unroll
            for (int i = 0; i < 6; ++i) {
                const int y = __shfl_up_sync(0xffffffffu, P[i], d, 8);
                if ((lane & 7) >= d) P[i] += y;
            }
    }
#endif
    unsigned long long d0 = 0, d1 = 0, d2 = 0;
    for (int j = threadIdx.x; j < SREC_B; j += NT) S.won[j] = 0xFFFFFFFFu;
    unsigned int stamp = 0;   // group counter of the cached path (won flags)
    __syncthreads();

    for (int c = c_begin + z; c < c_end; c += t.splits) {
        const Chunk ch = t.chunks[c];
        const size_t bi = (size_t)c * t.T + tile;
        const long long o = t.off[bi];
        const int n = (int)(t.off[bi + 1] - o);
        if (n == 0) continue;
        BinCtx bc;
        bc.status = t.status;
        bc.rseg = t.rec + (size_t)(rec_off + (long long)ch.s * t.F) * REC_F4;
        bc.key0 = t.key + im.key_off + (size_t)ch.s * t.V;
        bc.key1 = bc.key0 + t.V;
        bc.fcol = t.fcol;
        bc.ent = t.entries + o;
        bc.n = n;
        bc.fb = o + n > t.cap;
        if (MODE == 0 && t.vis && !bc.fb && n <= VIS_MAXN) {
            if (t.vis_gathered) continue;   // taken by k6v_raster_bwd (k_gather.cu)
            // visibility from the forward's buffer (BLUR_CACHE_VISIBILITY): the pixels add their moments
            // to the slots they name, only the (face, sub-frame) pairs that won are staged
            const int Gs = min(GMAX_B, group_div(SREC_B, n));
            FaceAcc acc;
            acc_zero(acc);
            for (int kg = ch.k0; kg < ch.k1; kg += Gs) {
                const int ng = min(Gs, ch.k1 - kg);
                ++stamp;
                if (threadIdx.x < ng) S.taus[threadIdx.x] = t.sched_tau[sched_off + kg + threadIdx.x];
                const uint16_t *vrow = t.vis + ((size_t)(im.cov_off + kg) * t.T + tile) * (TW * TH) + myp;
                const int4 q = S.qg[myp];
                for (int l = 0; l < ng; ++l, vrow += (size_t)t.T * (TW * TH)) {
                    const uint16_t v = *vrow;
                    if (inimg && v != 0xFFFF) {
                        S.won[l * n + v] = stamp;
                        add_moments(S.imom[l * n + v], q, dx, dy);
                    }
                }
                __syncthreads();
                stage_won(bc, n, S.taus, ng, tc, t.F, S.won, stamp, S.rec);
                __syncthreads();
                for (int j = threadIdx.x; j < n; j += NT) {   // one thread per bin slot
                    for (int l = 0; l < ng; ++l) {
                        float m[9];
                        if (take_moments(S.imom[l * n + j], inv_scale, tc.sx, tc.sy, m) == 0) continue;
                        float dv[6], dcl[9];
                        face_grad(S.rec[l * n + j], m, t.fcol, dv, dcl);
                        const float tau = S.taus[l];
                        if (j == (int)threadIdx.x) {
#pragma unroll
                            for (int i = 0; i < 6; ++i) {
                                acc.k0[i] = __fmaf_rn(1.f - tau, dv[i], acc.k0[i]);
                                acc.k1[i] = __fmaf_rn(tau, dv[i], acc.k1[i]);
                            }
#pragma unroll
                            for (int i = 0; i < 9; ++i) acc.c[i] += dcl[i];
                        } else {
                            float a0[6], a1[6];
#pragma unroll
                            for (int i = 0; i < 6; ++i) { a0[i] = (1.f - tau) * dv[i]; a1[i] = tau * dv[i]; }
                            flush(t, im, ch.s, S.rec[l * n + j].fid, a0, a1, dcl, dC);
                        }
                    }
                }
                __syncthreads();
            }
            if ((int)threadIdx.x < n) {
                bool nz = false;
#pragma unroll
                for (int i = 0; i < 9; ++i) nz |= acc.c[i] != 0.f;
#pragma unroll
                for (int i = 0; i < 6; ++i) nz |= (acc.k0[i] != 0.f) | (acc.k1[i] != 0.f);
                if (nz) flush(t, im, ch.s, __ldg(bc.ent + threadIdx.x), acc.k0, acc.k1, acc.c, dC);
            }
        } else if (!bc.fb && n <= SREC_B) {
            const int Gs = min(GMAX_B, group_div(SREC_B, n)), nw = (n + 31) >> 5;
            FaceAcc acc;
            acc_zero(acc);
            for (int kg = ch.k0; kg < ch.k1; kg += Gs) {
                const int ng = min(Gs, ch.k1 - kg);
                clear_words(S.wm, ng * NFP * nw);
                if (threadIdx.x < ng) S.taus[threadIdx.x] = t.sched_tau[sched_off + kg + threadIdx.x];
                __syncthreads();
                stage_group<false, MODE, true>(bc, n, 0, S.taus, ng, tc, t.W, t.H, t.F, S.sid, S.rec, S.vtx, S.wm, d2);
                __syncthreads();
                const int4 q = S.qg[myp];
                for (int l = 0; l < ng; ++l) {       // visibility, then the pixel's moments (no barriers)
                    float zbest = __int_as_float(0x7f800000);
                    int ebest = -1, fbest = 0x7fffffff;
                    const uint32_t *wml = S.wm + (l * NFP + fp_of(warp, lane)) * nw;
                    bool tie = true;
                    if (MODE != 2) tie = vis_mask_fast<false, MODE>(S.rec + l * n, wml, nw, ul, vl, zbest, ebest, d0, d1, false);
                    if (__any_sync(0xffffffffu, tie)) {
                        zbest = __int_as_float(0x7f800000);
                        ebest = -1;
                        vis_mask<false, MODE>(S.rec + l * n, S.vtx + 3 * l * n, wml, nw, 0, ul, vl, zbest, ebest, fbest,
                                              d0, d1, false);
                    }
#if BR_FX_RUNS
                    run_moments(&S.imom[0][0], (inimg && ebest >= 0) ? l * n + ebest : -1, lane, P, dy);
#else
                    if (inimg && ebest >= 0) add_moments(S.imom[l * n + ebest], q, dx, dy);
#endif
                }
                __syncthreads();
                for (int j = threadIdx.x; j < n; j += NT) {   // one thread per bin slot
                    for (int l = 0; l < ng; ++l) {
                        float m[9];
                        if (take_moments(S.imom[l * n + j], inv_scale, tc.sx, tc.sy, m) == 0) continue;
                        float dv[6], dcl[9];
                        face_grad(S.rec[l * n + j], m, t.fcol, dv, dcl);
                        const float tau = S.taus[l];
                        if (j == (int)threadIdx.x) {
#pragma unroll
                            for (int i = 0; i < 6; ++i) {
                                acc.k0[i] = __fmaf_rn(1.f - tau, dv[i], acc.k0[i]);
                                acc.k1[i] = __fmaf_rn(tau, dv[i], acc.k1[i]);
                            }
#pragma unroll
                            for (int i = 0; i < 9; ++i) acc.c[i] += dcl[i];
                        } else {
                            float a0[6], a1[6];
#pragma unroll
                            for (int i = 0; i < 6; ++i) { a0[i] = (1.f - tau) * dv[i]; a1[i] = tau * dv[i]; }
                            flush(t, im, ch.s, S.rec[l * n + j].fid, a0, a1, dcl, dC);
                        }
                    }
                }
                __syncthreads();
            }
            if ((int)threadIdx.x < n) {   // persistent slot of this thread
                bool nz = false;
#pragma unroll
                for (int i = 0; i < 9; ++i) nz |= acc.c[i] != 0.f;
#pragma unroll
                for (int i = 0; i < 6; ++i) nz |= (acc.k0[i] != 0.f) | (acc.k1[i] != 0.f);
                if (nz) flush(t, im, ch.s, __ldg(bc.ent + threadIdx.x), acc.k0, acc.k1, acc.c, dC);
            }
        } else {
            for (int k = ch.k0; k < ch.k1; ++k) {
                const float tau = t.sched_tau[sched_off + k];
                float zbest = __int_as_float(0x7f800000);
                int ebest = -1, fbest = 0x7fffffff;
                int base = 0, fpos = 0;
                if (threadIdx.x == 0) S.taus[0] = tau;
                while (true) {                         // visibility over all batches
                    const int nb = next_batch(bc, t.F, tau, tc, t.W, t.H, SREC_B, base, fpos, S.sid, S.wsum);
                    if (nb == 0) break;
                    const int nw = (nb + 31) >> 5;
                    clear_words(S.wm, NFP * nw);
                    __syncthreads();
                    stage_group<false, MODE, true>(bc, nb, base, S.taus, 1, tc, t.W, t.H, t.F, S.sid, S.rec, S.vtx, S.wm, d2);
                    __syncthreads();
                    vis_mask<false, MODE>(S.rec, S.vtx, S.wm + fp_of(warp, lane) * nw, nw, base, ul, vl, zbest, ebest, fbest, d0, d1,
                                          false);
                    if (ebest >= base) fbest = S.rec[ebest - base].fid;
                    base += nb;
                    __syncthreads();
                }
                if (!inimg) ebest = -1;
                base = 0;
                fpos = 0;
                while (true) {                         // re-stage each batch, moments and gradients of its winners
                    const int nb = next_batch(bc, t.F, tau, tc, t.W, t.H, SREC_B, base, fpos, S.sid, S.wsum);
                    if (nb == 0) break;
                    const int nw = (nb + 31) >> 5;
                    clear_words(S.wm, NFP * nw);
                    __syncthreads();
                    stage_group<false, MODE, true>(bc, nb, base, S.taus, 1, tc, t.W, t.H, t.F, S.sid, S.rec, S.vtx, S.wm, d2);
                    __syncthreads();
#if BR_FX_RUNS
                    run_moments(&S.imom[0][0], (ebest >= base && ebest < base + nb) ? ebest - base : -1, lane, P, dy);
#else
                    if (ebest >= base && ebest < base + nb) add_moments(S.imom[ebest - base], S.qg[myp], dx, dy);
#endif
                    __syncthreads();
                    for (int j = threadIdx.x; j < nb; j += NT) {
                        float m[9];
                        if (take_moments(S.imom[j], inv_scale, tc.sx, tc.sy, m) == 0) continue;
                        float dv[6], dcl[9], a0[6], a1[6];
                        face_grad(S.rec[j], m, t.fcol, dv, dcl);
#pragma unroll
                        for (int i = 0; i < 6; ++i) { a0[i] = (1.f - tau) * dv[i]; a1[i] = tau * dv[i]; }
                        flush(t, im, ch.s, S.rec[j].fid, a0, a1, dcl, dC);
                    }
                    base += nb;
                    __syncthreads();
                }
            }
        }
    }
}

template <bool CENSUS, int MODE>
static cudaError_t launch_fwd_t(const Tables &t, float *out, int *ids, int ids_k, unsigned long long *census,
                                cudaStream_t st)
{
    dim3 grid(t.T, t.B, t.splits);
    const int smem = (int)sizeof(FwdSmem<MODE>);
    cudaError_t e = cudaFuncSetAttribute(k4_raster_fwd<CENSUS, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    k4_raster_fwd<CENSUS, MODE><<<grid, NT, smem, st>>>(t, out, ids, ids_k, census);
    return cudaGetLastError();
}

template <int MODE>
static cudaError_t launch_bwd_t(const Tables &t, const float *grad, float *dC, cudaStream_t st)
{
    dim3 grid(t.T, t.B, t.splits);
#ifdef BR_K6_SORT
    if (!t.vis) {   // round 1's float counting-sort gather for the cached path (A/B: 6.86 vs 6.92 ms on C4)
#else
    if (true) {     // fixed-point moments (k6_raster_bwd_fx), visibility cached or recomputed: both paths
                    // reduce the same integer moments
#endif
        const int smem = (int)sizeof(BwdFxSmem<MODE>);
        cudaError_t e = cudaFuncSetAttribute(k6_raster_bwd_fx<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        if (t.vis_gathered)   // grid-stride over the listed (image, tile)s
            grid = dim3((unsigned)std::min<long long>((long long)t.T * t.B, 148LL * BR_K6_MINB), 1, t.splits);
        k6_raster_bwd_fx<MODE><<<grid, NT, smem, st>>>(t, grad, dC);
        return cudaGetLastError();
    }
    const int smem = (int)sizeof(BwdSmem<MODE>);
    cudaError_t e = cudaFuncSetAttribute(k6_raster_bwd<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    k6_raster_bwd<MODE><<<grid, NT, smem, st>>>(t, grad, dC);
    return cudaGetLastError();
}

// out = sum over splits of the partial images, in split order (deterministic)
__global__ void __launch_bounds__(256) k_split_reduce(const float4 *__restrict__ part, float4 *__restrict__ out,
                                                      size_t n, int splits)
{
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        float4 a = part[i];
        for (int z = 1; z < splits; ++z) {
            const float4 b = part[(size_t)z * n + i];
            a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
        }
        out[i] = a;
    }
}

cudaError_t launch_split_reduce(const Tables &t, float *out, cudaStream_t st)
{
    const size_t n = (size_t)t.B * t.H * t.W;
    if (n == 0) return cudaSuccess;
    const unsigned blocks = (unsigned)std::min<size_t>((n + 255) / 256, 148 * 16);
    k_split_reduce<<<blocks, 256, 0, st>>>(t.part, reinterpret_cast<float4 *>(out), n, t.splits);
    return cudaGetLastError();
}

cudaError_t launch_raster_fwd_legacy(const Tables &t, float *out, int *ids, int ids_k, unsigned long long *census,
                                     cudaStream_t st)
{
    if (t.B == 0 || t.T == 0) return cudaSuccess;
    switch (t.solver * 2 + (census ? 1 : 0)) {
    case 0:
        if (pixmajor_fwd_on()) return launch_raster_fwd_pixmajor(t, out, ids, ids_k, st);
        if (pipe_fwd_on())
            return t.covbits ? launch_fwd_pipe<true>(t, out, ids, ids_k, st) : launch_fwd_pipe<false>(t, out, ids, ids_k, st);
        if (sg_fwd_on())
            return t.covbits ? launch_fwd_sg<true>(t, out, ids, ids_k, st) : launch_fwd_sg<false>(t, out, ids, ids_k, st);
        if (!lean_fwd_off())
            return t.covbits ? launch_fwd_lean<true>(t, out, ids, ids_k, st) : launch_fwd_lean<false>(t, out, ids, ids_k, st);
        return launch_fwd_t<false, 0>(t, out, ids, ids_k, nullptr, st);
    case 1: {   // census: the algorithmic counts (every bin face tested), then the timed kernel's own counts
        cudaError_t e = launch_fwd_t<true, 0>(t, out, ids, ids_k, census, st);
        if (e != cudaSuccess || lean_fwd_off() || pipe_fwd_on()) return e;
        return t.covbits ? launch_fwd_lean<true, true>(t, out, ids, ids_k, st, census + 8)
                         : launch_fwd_lean<false, true>(t, out, ids, ids_k, st, census + 8);
    }
    case 2: return launch_fwd_t<false, 1>(t, out, ids, ids_k, nullptr, st);
    case 3: return launch_fwd_t<true, 1>(t, out, ids, ids_k, census, st);
    case 4: return launch_fwd_t<false, 2>(t, out, ids, ids_k, nullptr, st);
    default: return launch_fwd_t<true, 2>(t, out, ids, ids_k, census, st);
    }
}

// BLURRAST_VIS_GATHER=0: the cached chunks take k6_raster_bwd_fx's cached path instead (A/B)
static bool vis_gather_off()
{
    const char *s = std::getenv("BLURRAST_VIS_GATHER");
    return s && s[0] == '0';
}

cudaError_t launch_raster_bwd_legacy(const Tables &t, const float *grad, float *dC, cudaStream_t st)
{
    if (t.B == 0 || t.T == 0 || t.F == 0) return cudaSuccess;
    switch (t.solver) {
    case 0:
        if (t.vis && !vis_gather_off()) {   // cached chunks: visibility gather (k_gather.cu); the rest below
            cudaError_t e = launch_vis_gather(t, grad, dC, st);
            if (e != cudaSuccess) return e;
            Tables t2 = t;
            t2.vis_gathered = 1;
            return launch_bwd_t<0>(t2, grad, dC, st);
        }
        return launch_bwd_t<0>(t, grad, dC, st);
    case 1: return launch_bwd_t<1>(t, grad, dC, st);
    default: return launch_bwd_t<2>(t, grad, dC, st);
    }
}

}  // namespace br
