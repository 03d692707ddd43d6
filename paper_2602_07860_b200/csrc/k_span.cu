// k_span.cu -- K4 fused raster-forward and K6 fused raster-backward of the fast solver (solver 0):
// exact span rasterization of the staged (face, sub-frame) records into a shared-memory z-buffer.
//
// One CTA = one 16x16 pixel tile of one image (grid tiles x images x splits, as in k_raster.cu).  For
// each group of up to SP_GMAX sub-frames of a chunk (one bin of faces, K3):
//   stage+walk  one thread per (bin face j, sub-frame tau_l): the (face, segment) coefficient record is
//               evaluated at tau by Horner (Eq.8's numerators and denominator, "computed only once" per
//               segment), sign-normalised by det F(tau) and re-centred at the tile centre; the
//               same thread then walks the rows of the face's per-tau pixel box.  In a row v the three
//               edge functions e_i(x) = fma(A_i, u(x), fma(B_i, v, G_i)) -- the numerators N_i of Eq.8 up to
//               the positive factor 1/|D| -- are monotone in x (a correctly rounded fma of an increasing
//               u(x)), so the covered pixels (all w_i >= 0) form one interval.  Its ends come from
//               each edge's boundary x = TW/2 - R_i / (A_i sx); where a boundary lies within SPAN_DLT px of a
//               pixel centre the end pixel is re-tested with exactly the per-pixel arithmetic, so the span
//               is the exact covered set of the per-pixel fp32 test (the same decisions as k_raster.cu).
//               Each covered pixel offers the key (order(depth) << 32 | face id << 10 | slot) to the
//               sub-frame's z-buffer by a 64-bit shared-memory compare-and-swap min: the lexicographic
//               (depth, face index) z-test of Q7 (strict < on depth, the lower face index wins exact ties).
//               No pixel is tested against a face that does not cover it.
//   resolve     one thread per pixel: the winner of every sub-frame of the group is read back (and the
//               z-buffer entry reset); fwd: w_i = N_i/|D|, I = sum w_i c_i (Eq.9) accumulated in registers over
//               all sub-frames -- the sub-frames never reach HBM; bwd: see k6s_raster_bwd.
// Bins longer than the record stage, and overflowed bins (exact rescan of all faces, status
// EOVERFLOW), are processed per sub-frame in batches that share the sub-frame's z-buffer.
#include <algorithm>
#include <cstdio>

#include "internal.cuh"
#include "raster_common.cuh"
#include "../../include/blurrast.h"

namespace br {

#ifndef BR_SP_SREC_F
#define BR_SP_SREC_F 256
#endif
#ifndef BR_SP_SREC_B
#define BR_SP_SREC_B 256
#endif
#ifndef BR_SP_GMAX
#define BR_SP_GMAX 8
#endif
#ifndef BR_SP_GMAX_B
#define BR_SP_GMAX_B 4
#endif
#ifndef BR_SP_MINB_F
#define BR_SP_MINB_F 4
#endif
#ifndef BR_SP_MINB_B
#define BR_SP_MINB_B 4
#endif
constexpr int SP_SREC_F = BR_SP_SREC_F;   // fwd: staged (face, sub-frame) records per CTA
constexpr int SP_SREC_B = BR_SP_SREC_B;   // bwd
constexpr int SP_GMAX = BR_SP_GMAX;       // fwd: sub-frames staged together (z-buffer layers)
constexpr int SP_GMAX_B = BR_SP_GMAX_B;   // bwd
static_assert(SP_SREC_F <= 1024 && SP_SREC_B <= 1024, "slot field of the z-buffer key is 10 bits");
constexpr unsigned long long ZB_EMPTY = ~0ull;
constexpr float SPAN_DLT = 1.0f / 1024.0f;   // px: boundaries closer than this to a pixel centre are re-tested

struct __align__(16) SpanRec {   // a (face, sub-frame) record for this tile, 64 B
    float a[3], b[3], g[3];      // sign-normalised edge functions e_i = a_i ul + b_i vl + g_i (tile-local)
    float invD;                  // 1 / |det F(tau)|
    int fid;
    int box;                     // x0 | x1 << 4 | y0 << 8 | y1 << 12 (tile-local pixel box) | l << 16 (sub-frame
                                 // layer) | first run << 20; -1: no record
    float az, bz, cz;            // depth plane z = fma(az, ul, fma(bz, vl, cz)) (Q6)
    unsigned tag;                // z-buffer key low word: fid << 10 | slot j
};
static_assert(SP_GMAX <= 16, "layer field of SpanRec::box is 4 bits");
static_assert(SP_SREC_F * TH <= 4096 && SP_SREC_B * TH <= 4096, "run index field of SpanRec::box is 12 bits");
// a run: the exact covered pixels [lo, hi] of row y of record r: r << 12 | y << 8 | lo << 4 | hi (lo > hi: none)
__device__ __forceinline__ unsigned run_word(int r, int y, int lo, int hi)
{
    return lo <= hi ? ((unsigned)r << 12) | ((unsigned)y << 8) | ((unsigned)lo << 4) | (unsigned)hi
                    : ((unsigned)r << 12) | ((unsigned)y << 8) | 0x10u;   // lo = 1, hi = 0
}

// order-preserving map of a float onto uint32 (for the depth half of the z-buffer key)
__device__ __forceinline__ unsigned zord(float z)
{
    const unsigned u = __float_as_uint(z);
    return u ^ ((unsigned)((int)u >> 31) | 0x80000000u);
}

__device__ __forceinline__ void zmin(unsigned long long *p, unsigned long long v)
{
    unsigned long long old = *(volatile unsigned long long *)p;
    while (v < old) {
        const unsigned long long prev = atomicCAS(p, old, v);
        if (prev == old) break;
        old = prev;
    }
}

// The per-pixel coverage test of the fast path: all three sign-normalised edge functions >= 0 at the
// pixel centre (R_i = fma(B_i, vl, G_i) of the row).
__device__ __forceinline__ bool cov_at(const float A[3], const float R[3], int x, float sx)
{
    const float ul = (float)(x - TW / 2) * sx;
    return fminf(fminf(__fmaf_rn(A[0], ul, R[0]), __fmaf_rn(A[1], ul, R[1])), __fmaf_rn(A[2], ul, R[2])) >= 0.f;
}

// Exact covered range of row y (tile-local x within [x0, x1]; lo > hi: none).
//
// Every edge function e_i(x) = fma(A_i, ul(x), R_i) of the row is monotone in x (a correctly rounded fma
// of an increasing ul(x)), so the covered pixels form one interval, bounded below by the edges with
// A_i > 0 and above by those with A_i < 0; an edge's boundary is x* = TW/2 - R_i / (A_i sx).  The record
// carries these boundaries as lines in y (fast form, accurate to < 3e-4 px) -- or, for SLOW records (an
// edge steeper than 500 px per row, |A_i sx| underflowing, three same-side edges), the row evaluates them
// from R_i and k_i = -1/(A_i sx) -- and a range end that lies within SPAN_DLT of a pixel centre is
// re-tested with the per-pixel arithmetic itself, scanning inward.  The result is exactly the set of
// pixels of the row that pass cov_at.  Returns the number of exact tests taken (census).
__device__ __forceinline__ int row_range(const float ln[8], bool slow, const SpanRec &Rec, int y, int x0, int x1,
                                         const TileCtx &tc, int &lo, int &hi)
{
    float L, U;
    bool force = false;
    if (!slow) {
        const float yf = (float)y;
        L = fmaxf(fmaf(ln[1], yf, ln[0]), fmaf(ln[3], yf, ln[2]));
        U = fminf(fmaf(ln[5], yf, ln[4]), fmaf(ln[7], yf, ln[6]));
    } else {   // per-edge boundaries from the row's exact R_i
        const float vl = (float)(TH / 2 - y) * tc.sy;
        L = -1000.5f;
        U = 1000.5f;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            const float A = Rec.a[i], R = __fmaf_rn(Rec.b[i], vl, Rec.g[i]);
            const float as = A * tc.sx;
            if (fabsf(as) >= 1e-30f) {
                const float t = fminf(fmaxf(fmaf(R, -__frcp_rn(as), (float)(TW / 2)), -100.5f), 116.5f);
                if (A > 0.f) L = fmaxf(L, t); else U = fminf(U, t);
            } else if (A != 0.f) {
                force = true;                  // no usable bound: the ends are scanned inward exactly
            } else if (R < 0.f) {
                U = -1000.5f;                  // e_i = R_i < 0 on the whole row
            }
        }
    }
    const float cl = ceilf(L - SPAN_DLT), ch = floorf(U + SPAN_DLT);
    lo = max((int)cl, x0);
    hi = min((int)ch, x1);
    int nt = 0;
    if (lo <= hi && (force || cl <= L + SPAN_DLT || ch >= U - SPAN_DLT)) {
        // a range end within SPAN_DLT of a boundary: move the ends inward with the exact test
        const float vl = (float)(TH / 2 - y) * tc.sy;
        const float A[3] = {Rec.a[0], Rec.a[1], Rec.a[2]};
        const float R[3] = {__fmaf_rn(Rec.b[0], vl, Rec.g[0]), __fmaf_rn(Rec.b[1], vl, Rec.g[1]),
                            __fmaf_rn(Rec.b[2], vl, Rec.g[2])};
        while (lo <= hi && !cov_at(A, R, lo, tc.sx)) { ++lo; ++nt; }
        while (lo <= hi && !cov_at(A, R, hi, tc.sx)) { --hi; ++nt; }
        nt += lo <= hi ? 2 : 0;
    }
    return nt;
}

// Evaluate a (face, segment) record at tau for this tile (the arithmetic of k_raster.cu's stage_tau):
// sign-normalised edge functions, 1/|D| and the depth plane z(ul, vl) = fma(az, ul, fma(bz, vl, cz)),
// the screen-space interpolation of the view depth (Q6) written as z0 + w1 (z1 - z0) + w2 (z2 - z0).
__device__ __forceinline__ void eval_tau(const FaceRec &fr, float tau, float D, const TileCtx &tc, float A[3],
                                         float B[3], float G[3], float &invD, float &az, float &bz, float &cz)
{
    const float sg = D < 0.f ? -1.f : 1.f;
    invD = 1.0f / fabsf(D);
    const float *ef = reinterpret_cast<const float *>(fr.q);
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const float ox = ef[8 * i], oy = ef[8 * i + 1];
        const float al = __fmaf_rn(tau, ef[8 * i + 3], ef[8 * i + 2]);
        const float be = __fmaf_rn(tau, ef[8 * i + 5], ef[8 * i + 4]);
        const float ga = __fmul_rn(tau, __fmaf_rn(tau, ef[8 * i + 7], ef[8 * i + 6]));
        const float dx = __fsub_rn(tc.uc, ox), dy = __fsub_rn(tc.vc, oy);
        const float gp = __fmaf_rn(al, dx, __fmaf_rn(be, dy, ga));
        A[i] = al * sg;
        B[i] = be * sg;
        G[i] = gp * sg;
    }
    const float4 z0 = fr.q[9], z1 = fr.q[10];
    const float za = __fmaf_rn(tau, z1.x - z0.x, z0.x);
    const float zb = __fmaf_rn(tau, z1.y - z0.y, z0.y);
    const float zc = __fmaf_rn(tau, z1.z - z0.z, z0.z);
    const float dzb = zb - za, dzc = zc - za;
    az = __fmaf_rn(A[1], dzb, A[2] * dzc) * invD;
    bz = __fmaf_rn(B[1], dzb, B[2] * dzc) * invD;
    cz = __fmaf_rn(__fmaf_rn(G[1], dzb, G[2] * dzc), invD, za);
}

// Boundary lines of the record (see row_range) and the exact row range of the edges with A_i == 0
// (e_i = R_i does not depend on x: rows with R_i < 0 are dropped from [y0, y1]).  Returns false when no
// row is left.  slow: the lines are not used (see row_range).
__device__ __forceinline__ bool span_lines(const float A[3], const float B[3], const float G[3], const TileCtx &tc,
                                           int &y0, int &y1, float ln[8], bool &slow)
{
    int nl = 0, nu = 0;
    slow = false;
    float l0 = -1000.5f, l1 = 0.f, l2 = -1000.5f, l3 = 0.f, u0 = 1000.5f, u1 = 0.f, u2 = 1000.5f, u3 = 0.f;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        if (A[i] == 0.f) {
            while (y0 <= y1 && __fmaf_rn(B[i], (float)(TH / 2 - y0) * tc.sy, G[i]) < 0.f) ++y0;
            while (y0 <= y1 && __fmaf_rn(B[i], (float)(TH / 2 - y1) * tc.sy, G[i]) < 0.f) --y1;
            continue;
        }
        // x*(y) = TW/2 - (B_i vl(y) + G_i) / (A_i sx), vl(y) = (TH/2 - y) sy: each term carries a few ulp
        // of relative error, so lines with |T0| + 16 |TY| < 500 px are accurate to < 3e-4 px (< SPAN_DLT)
        const float as = A[i] * tc.sx;
        const float k = -__frcp_rn(as);
        const float bs = B[i] * tc.sy;
        const float f0 = fmaf(k, fmaf(bs, (float)(TH / 2), G[i]), (float)(TW / 2)), f1 = -k * bs;
        if (!(fabsf(f0) + 16.f * fabsf(f1) < 500.f) || !(fabsf(as) >= 1e-30f)) slow = true;
        if (A[i] > 0.f) {
            if (nl == 0) { l0 = f0; l1 = f1; } else if (nl == 1) { l2 = f0; l3 = f1; } else slow = true;
            ++nl;
        } else {
            if (nu == 0) { u0 = f0; u1 = f1; } else if (nu == 1) { u2 = f0; u3 = f1; } else slow = true;
            ++nu;
        }
    }
    ln[0] = l0; ln[1] = l1; ln[2] = l2; ln[3] = l3; ln[4] = u0; ln[5] = u1; ln[6] = u2; ln[7] = u3;
    return y0 <= y1;
}

__device__ __forceinline__ void store_rec(SpanRec &o, const float A[3], const float B[3], const float G[3], float invD,
                                          int fid, int box, float az, float bz, float cz, unsigned tag)
{
    float4 *q = reinterpret_cast<float4 *>(&o);
    q[0] = make_float4(A[0], A[1], A[2], B[0]);
    q[1] = make_float4(B[1], B[2], G[0], G[1]);
    q[2] = make_float4(G[2], invD, __int_as_float(fid), __int_as_float(box));
    q[3] = make_float4(az, bz, cz, __uint_as_float(tag));
}

struct WalkCount {
    unsigned long long frag = 0, test = 0, rec = 0;
};

// Stage the bin faces [base, base+nb) (or sid[] on the fallback path) at the ng sub-frames taus[0..ng):
// one thread per (face j, sub-frame l) pair builds the record rec[l * nb + j] and the exact covered
// range of every row of its pixel box (row_range), written as run words to runs[] (one slot per box row,
// reserved with one shared atomic per warp).  Pairs without coverage get box = -1.  Work is spread
// face-major, so lanes sharing a face load its (face, segment) record with broadcast loads.
template <bool CENSUS>
__device__ __forceinline__ void stage_runs(const BinCtx &bc, int nb, int base, const float *taus, int ng,
                                           const TileCtx &tc, int W, int H, int F, const int *sid, SpanRec *rec,
                                           unsigned *runs, int *nruns, WalkCount &wc)
{
    const int lane = threadIdx.x & 31;
    const float inv_ng = 1.0f / (float)ng;
    const int npair = nb * ng;
    for (int p0 = 0; p0 < npair; p0 += NT) {   // block-uniform trip count: the warp scan below is convergent
        const int p = p0 + threadIdx.x;
        int rows = 0, y0 = 0, r = 0, x0 = 0, x1 = -1, y1 = -1;
        bool slow = false;
        float ln[8];
        SpanRec *out = nullptr;
        int box = 0;
        if (p < npair) {
            const int j = div_small(p, inv_ng), l = p - j * ng;
            r = l * nb + j;
            out = rec + r;
            out->box = -1;
            const int f = bc.fb ? sid[j] : __ldg(bc.ent + base + j);
            if ((unsigned)f >= (unsigned)F) {     // never expected: bins hold valid face ids
                atomicOr(bc.status, BLUR_ST_EINTERNAL);
            } else {
                const float4 *rp = bc.rseg + (size_t)f * REC_F4;
                const float4 q6 = __ldg(rp + 6);
                const float tau = taus[l];
                const float D = __fmaf_rn(tau, __fmaf_rn(tau, q6.x, q6.y), q6.z);   // det F(tau), A8
                bool ok = __float_as_int(q6.w) >= 0 && fabsf(D) > EPS_D;          // skipped face; Q8
                if (ok) {
                    const float4 b0 = __ldg(rp + 7), b1 = __ldg(rp + 8);
                    ok = tile_pixels(box_lerp(tau, b0.x, b1.x), box_lerp(tau, b0.y, b1.y), box_lerp(tau, b0.z, b1.z),
                                     box_lerp(tau, b0.w, b1.w), W, H, tc, x0, x1, y0, y1);
                }
                if (ok) {
                    FaceRec fr;
                    load_rec(rp, fr);
                    float A[3], B[3], G[3], invD, az, bz, cz;
                    eval_tau(fr, tau, D, tc, A, B, G, invD, az, bz, cz);
                    if (span_lines(A, B, G, tc, y0, y1, ln, slow)) {
                        const int fid = __float_as_int(q6.w);
                        box = x0 | (x1 << 4) | (y0 << 8) | (y1 << 12) | (l << 16);
                        store_rec(*out, A, B, G, invD, fid, box, az, bz, cz, ((unsigned)fid << 10) | (unsigned)j);
                        rows = y1 - y0 + 1;
                        if (CENSUS) wc.rec++;
                    }
                }
            }
        }
        int incl = rows;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        const int tot = __shfl_sync(0xffffffffu, incl, 31);
        int b0 = 0;
        if (lane == 31 && tot > 0) b0 = atomicAdd(nruns, tot);
        b0 = __shfl_sync(0xffffffffu, b0, 31) + incl - rows;
        if (rows > 0) out->box = box | (b0 << 20);
        for (int k = 0; k < rows; ++k) {
            int lo, hi;
            const int nt = row_range(ln, slow, *out, y0 + k, x0, x1, tc, lo, hi);
            if (CENSUS) { wc.test += nt; wc.frag += hi >= lo ? hi - lo + 1 : 0; }
            runs[b0 + k] = run_word(r, y0 + k, lo, hi);
        }
    }
}

// Walk the runs[0..nr): the covered pixels of each warp's 32 runs are spread evenly over its lanes
// (rounds of 32 pixels: each lane finds the run its pixel belongs to from the runs' start positions in
// the round and takes the run's data by shuffles), and every covered pixel offers its key
// (order(depth) << 32 | fid << 10 | slot j) to the z-buffer layer of the record's sub-frame (64-bit
// shared CAS min).  win: 32 ints per warp.
__device__ __forceinline__ void walk_runs(const SpanRec *rec, const unsigned *runs, int nr, const TileCtx &tc,
                                          unsigned long long *zb, int *wwin)
{
    const int lane = threadIdx.x & 31;
    int *win = wwin + (threadIdx.x >> 5) * 32;
    for (int u0 = 0; u0 < nr; u0 += NT) {   // block-uniform trip count (the warp collectives are convergent)
        const int u = u0 + (int)threadIdx.x;
        int lo = 0, cnt = 0, zoff = 0;
        float az = 0.f, rz = 0.f;
        unsigned tag = 0;
        if (u < nr) {
            const unsigned w = runs[u];
            lo = (w >> 4) & 15;
            cnt = max((int)(w & 15) - lo + 1, 0);
            if (cnt > 0) {
                const int r = (int)(w >> 12), y = (int)((w >> 8) & 15);
                const SpanRec &R = rec[r];
                const float4 zq = reinterpret_cast<const float4 *>(&R)[3];
                const float vl = (float)(TH / 2 - y) * tc.sy;
                az = zq.x;
                rz = __fmaf_rn(zq.y, vl, zq.z);
                tag = __float_as_uint(zq.w);
                zoff = ((R.box >> 16) & 15) * (TW * TH) + y * TW;
            }
        }
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        const int tot = __shfl_sync(0xffffffffu, incl, 31);
        const int excl = incl - cnt;
        for (int f0 = 0; f0 < tot; f0 += 32) {
            // runs starting in this round mark their start position; the other pixels of the round belong
            // to the last run started before it (the carried one)
            const bool st = cnt > 0 && excl >= f0 && excl < f0 + 32;
            if (st) win[excl - f0] = lane;
            const unsigned P = __reduce_or_sync(0xffffffffu, st ? 1u << (excl - f0) : 0u);
            const unsigned carry = __ballot_sync(0xffffffffu, cnt > 0 && excl < f0);
            __syncwarp();
            const unsigned le = P & (0xffffffffu >> (31 - lane));
            const int owner = le ? win[31 - __clz(le)] : 31 - __clz(carry);
            const int olo = __shfl_sync(0xffffffffu, lo, owner), oex = __shfl_sync(0xffffffffu, excl, owner);
            const float oaz = __shfl_sync(0xffffffffu, az, owner), orz = __shfl_sync(0xffffffffu, rz, owner);
            const unsigned otag = __shfl_sync(0xffffffffu, tag, owner);
            const int ozoff = __shfl_sync(0xffffffffu, zoff, owner);
            const int f = f0 + lane;
            if (f < tot) {
                const int x = olo + f - oex;
                const float ul = (float)(x - TW / 2) * tc.sx;
                const float z = __fmaf_rn(oaz, ul, orz);
                zmin(zb + ozoff + x, ((unsigned long long)zord(z) << 32) | otag);
            }
            __syncwarp();
        }
    }
}

struct SpFwdSmem {
    SpanRec rec[SP_SREC_F];
    unsigned long long zb[SP_GMAX][TW * TH];
    unsigned runs[SP_SREC_F * TH];   // covered row ranges of the group's records (run_word)
    int sid[SP_SREC_F];
    float taus[SP_GMAX];
    int wsum[NWARP];
    int nruns;
    int win[NWARP * 32];   // walk_runs: per-warp owner windows
    float4 acc[TW * TH];   // per-pixel (r, g, b, a) sums over the sub-frames (thread-private slot)
};

template <bool CENSUS>
__global__ void __launch_bounds__(NT, BR_SP_MINB_F) k4s_raster_fwd(Tables t, float *__restrict__ out,
                                                                  int *__restrict__ ids, int ids_k,
                                                                  unsigned long long *census)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SpFwdSmem &S = *reinterpret_cast<SpFwdSmem *>(smem_raw);
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
    const int myp = ly * TW + lx;
#define PIX (((size_t)b * t.H + py) * t.W + px)
    for (int l = 0; l < SP_GMAX; ++l) S.zb[l][threadIdx.x] = ZB_EMPTY;
    S.acc[myp] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (threadIdx.x == 0) S.nruns = 0;
    WalkCount wc;
    unsigned long long nshade = 0;
    __syncthreads();

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
        bc.key0 = bc.key1 = nullptr;
        bc.fcol = t.fcol;
        bc.ent = t.entries + o;
        bc.n = n;
        bc.fb = o + n > t.cap;
        if (!bc.fb && n <= SP_SREC_F) {
            // grouped path: the whole bin staged for up to Gs sub-frames at once
            const int Gs = min(SP_GMAX, group_div(SP_SREC_F, n));
            for (int kg = ch.k0; kg < ch.k1; kg += Gs) {
                const int ng = min(Gs, ch.k1 - kg);
                if (threadIdx.x < ng) S.taus[threadIdx.x] = t.sched_tau[sched_off + kg + threadIdx.x];
                __syncthreads();
                stage_runs<CENSUS>(bc, n, 0, S.taus, ng, tc, t.W, t.H, t.F, S.sid, S.rec, S.runs, &S.nruns, wc);
                __syncthreads();
                walk_runs(S.rec, S.runs, S.nruns, tc, &S.zb[0][0], S.win);
                __syncthreads();
                if (threadIdx.x == 0) S.nruns = 0;
                const float ul = (float)(lx - TW / 2) * tc.sx, vl = (float)(TH / 2 - ly) * tc.sy;
                for (int l = 0; l < ng; ++l) {
                    const unsigned long long key = S.zb[l][myp];
                    S.zb[l][myp] = ZB_EMPTY;
                    int fid = -1;
                    if (key != ZB_EMPTY) {
                        const SpanRec &r = S.rec[l * n + (int)(key & 1023u)];
                        float pr, pg, pb;
                        shade(r, t.fcol, ul, vl, pr, pg, pb);      // Eq.9
                        float4 a = S.acc[myp];
                        a.x += pr; a.y += pg; a.z += pb; a.w += 1.f;
                        S.acc[myp] = a;
                        fid = r.fid;
                        if (CENSUS) nshade++;
                    }
                    if (ids && inimg && kg + l == ids_k) ids[PIX] = fid;
                    if (t.covbits) {   // soft path: which pixels of the warp are covered at this sub-frame
                        const unsigned m = __ballot_sync(0xffffffffu, fid >= 0 || !inimg);
                        if (lane == 0) t.covbits[cov_word(t, im, kg + l, tile) + warp] = m;
                    }
                }
                __syncthreads();
            }
        } else {
            // per sub-frame, several batches (long bins) or the exact fallback scan (overflow); the
            // batches share the sub-frame's z-buffer layer 0, a winner is shaded when its batch is staged
            for (int k = ch.k0; k < ch.k1; ++k) {
                const float tau = t.sched_tau[sched_off + k];
                unsigned long long prev = ZB_EMPTY;
                int bfid = -1;
                float pr = 0.f, pg = 0.f, pb = 0.f;
                int base = 0, fpos = 0;
                if (threadIdx.x == 0) S.taus[0] = tau;
                while (true) {
                    const int nb = next_batch(bc, t.F, tau, tc, t.W, t.H, SP_SREC_F, base, fpos, S.sid, S.wsum);
                    if (nb == 0) break;
                    __syncthreads();
                    stage_runs<CENSUS>(bc, nb, base, S.taus, 1, tc, t.W, t.H, t.F, S.sid, S.rec, S.runs, &S.nruns, wc);
                    __syncthreads();
                    walk_runs(S.rec, S.runs, S.nruns, tc, &S.zb[0][0], S.win);
                    __syncthreads();
                    if (threadIdx.x == 0) S.nruns = 0;
                    const unsigned long long key = S.zb[0][myp];
                    if (key != prev) {   // the winner changed in this batch: shade it now (Eq.9)
                        const SpanRec &r = S.rec[(int)(key & 1023u)];
                        const float ul = (float)(lx - TW / 2) * tc.sx, vl = (float)(TH / 2 - ly) * tc.sy;
                        shade(r, t.fcol, ul, vl, pr, pg, pb);
                        bfid = r.fid;
                        prev = key;
                    }
                    base += nb;
                    __syncthreads();
                }
                S.zb[0][myp] = ZB_EMPTY;
                if (bfid >= 0) {
                    float4 a = S.acc[myp];
                    a.x += pr; a.y += pg; a.z += pb; a.w += 1.f;
                    S.acc[myp] = a;
                    if (CENSUS) nshade++;
                }
                if (ids && inimg && k == ids_k) ids[PIX] = bfid;
                if (t.covbits) {
                    const unsigned m = __ballot_sync(0xffffffffu, bfid >= 0 || !inimg);
                    if (lane == 0) t.covbits[cov_word(t, im, k, tile) + warp] = m;
                }
                __syncthreads();
            }
        }
    }
    if (inimg && out) {   // out == null: coverage-only pass (soft backward without a preceding forward)
        const float inv = 1.0f / (float)N;
        const float4 a = S.acc[myp];
        const float4 v = make_float4(a.x * inv, a.y * inv, a.z * inv, a.w * inv);
        if (t.splits == 1) reinterpret_cast<float4 *>(out)[PIX] = v;
        else t.part[(size_t)blockIdx.z * ((size_t)t.B * t.H * t.W) + PIX] = v;
    }
#undef PIX
    if (CENSUS) {
        atomicAdd(census + 0, wc.frag);
        atomicAdd(census + 1, nshade);
        atomicAdd(census + 2, wc.frag + wc.test);
        atomicAdd(census + 3, wc.rec);
    }
}

// ------------------------------------------------------------------ backward
//
// The z-buffer is rebuilt exactly as in the forward (stage_runs + walk_runs).  Then one thread per
// record (face j, sub-frame l) walks the record's rows again and sums the nine moments m = sum over its
// won pixels of g (1, u, v), g = dL/dI / N (the pixel's key names this face and slot), into the
// record's own shared slot (its boundary lines are not needed any more).  The face's gradient is linear
// in g and w_i(p) is affine in p, so (Eq.9, dw/dv_i = -w_i dw/dp; face_grad) the closed form gives
// dL/dc_i and the screen-space dL/dv_i(tau) from the moments.  One thread per bin face j then adds its
// records' gradients over the group's sub-frames, split (1 - tau, tau) onto the segment's keyframes
// (Eq.5-6), in registers across the chunk, and flushes one vector RED per (vertex, keyframe) and three
// per vertex colour at the end of the chunk.  No per-sub-frame data is stored in HBM: the winners are
// recomputed.

struct SpBwdSmem {
    SpanRec rec[SP_SREC_B];
    unsigned long long zb[SP_GMAX_B][TW * TH];
    unsigned runs[SP_SREC_B * TH];
    float mom[SP_SREC_B][10];   // per record: the nine moments of its won pixels and their count
    float4 g[TW * TH];          // dL/dI / N of the tile
    int sid[SP_SREC_B];
    float taus[SP_GMAX_B];
    int wsum[NWARP];
    int nruns;
    int win[NWARP * 32];
};

// moments of the pixels record r won (key low word == tag, or with by_fid (batched path: slots repeat
// across batches) key low word >> 10 == fid) over its runs, into mom[r]; returns the count
__device__ __forceinline__ int rec_moments(const SpanRec &R, const unsigned *runs, bool by_fid,
                                           const unsigned long long *zl, const float4 *g, const TileCtx &tc,
                                           float *mo)
{
    const int box = R.box;
    const int nrow = ((box >> 12) & 15) - ((box >> 8) & 15) + 1;
    const unsigned *rw = runs + ((unsigned)box >> 20);
    const unsigned tag = R.tag, fid = (unsigned)R.fid;
    float m[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) m[q] = 0.f;
    int cnt = 0;
    const unsigned *zw = reinterpret_cast<const unsigned *>(zl);
    for (int k = 0; k < nrow; ++k) {
        const unsigned w = rw[k];
        const int y = (w >> 8) & 15, lo = (w >> 4) & 15, hi = w & 15;
        const float vl = (float)(TH / 2 - y) * tc.sy;
        for (int x = lo; x <= hi; ++x) {
            const int p = y * TW + x;
            const unsigned kw = zw[2 * p];   // low word of the key (little-endian)
            if (by_fid ? (kw >> 10) == fid : kw == tag) {
                const float4 gg = g[p];
                const float ul = (float)(x - TW / 2) * tc.sx;
                m[0] += gg.x; m[1] += gg.y; m[2] += gg.z;
                m[3] += ul * gg.x; m[4] += ul * gg.y; m[5] += ul * gg.z;
                m[6] += vl * gg.x; m[7] += vl * gg.y; m[8] += vl * gg.z;
                ++cnt;
            }
        }
    }
#pragma unroll
    for (int q = 0; q < 9; ++q) mo[q] = m[q];
    mo[9] = __int_as_float(cnt);
    return cnt;
}

__global__ void __launch_bounds__(NT, BR_SP_MINB_B) k6s_raster_bwd(Tables t, const float *__restrict__ grad,
                                                                  float *__restrict__ dC)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SpBwdSmem &S = *reinterpret_cast<SpBwdSmem *>(smem_raw);
    const int b = blockIdx.y, tile = blockIdx.x;
    const ImgInfo &im = t.imgs[b];
    const int N = im.N, c_begin = im.chunk_begin, c_end = im.chunk_end, sched_off = im.sched_off;
    const long long rec_off = im.rec_off;
    TileCtx tc;
    tile_ctx(t, tile, tc);
    {
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        const int lx = (warp & 1) * 8 + (lane & 7), ly = (warp >> 1) * 4 + (lane >> 3);
        const int px = tc.px0 + lx, py = tc.py0 + ly;
        float4 g = make_float4(0.f, 0.f, 0.f, 0.f);
        if (px < t.W && py < t.H) {
            g = __ldg(reinterpret_cast<const float4 *>(grad) + ((size_t)b * t.H + py) * t.W + px);
            const float inv = 1.0f / (float)N;   // dI/dI_k = 1/N (uniform mean)
            g.x *= inv; g.y *= inv; g.z *= inv; g.w = 0.f;
        }
        S.g[ly * TW + lx] = g;
    }
    for (int l = 0; l < SP_GMAX_B; ++l) S.zb[l][threadIdx.x] = ZB_EMPTY;
    if (threadIdx.x == 0) S.nruns = 0;
    __syncthreads();
    WalkCount wc;

    for (int c = c_begin + (int)blockIdx.z; c < c_end; c += t.splits) {
        const Chunk ch = t.chunks[c];
        const size_t bi = (size_t)c * t.T + tile;
        const long long o = t.off[bi];
        const int n = (int)(t.off[bi + 1] - o);
        if (n == 0) continue;
        BinCtx bc;
        bc.status = t.status;
        bc.rseg = t.rec + (size_t)(rec_off + (long long)ch.s * t.F) * REC_F4;
        bc.key0 = bc.key1 = nullptr;
        bc.fcol = t.fcol;
        bc.ent = t.entries + o;
        bc.n = n;
        bc.fb = o + n > t.cap;
        if (!bc.fb && n <= SP_SREC_B) {
            const int Gs = min(SP_GMAX_B, group_div(SP_SREC_B, n));
            FaceAcc acc;
            acc_zero(acc);
            for (int kg = ch.k0; kg < ch.k1; kg += Gs) {
                const int ng = min(Gs, ch.k1 - kg);
                if (threadIdx.x < ng) S.taus[threadIdx.x] = t.sched_tau[sched_off + kg + threadIdx.x];
                __syncthreads();
                stage_runs<false>(bc, n, 0, S.taus, ng, tc, t.W, t.H, t.F, S.sid, S.rec, S.runs, &S.nruns, wc);
                __syncthreads();
                walk_runs(S.rec, S.runs, S.nruns, tc, &S.zb[0][0], S.win);
                __syncthreads();
                for (int r = threadIdx.x; r < n * ng; r += NT) {   // moments, one thread per record
                    const SpanRec &R = S.rec[r];
                    if (R.box < 0) { S.mom[r][9] = 0.f; continue; }
                    rec_moments(R, S.runs, false, &S.zb[(R.box >> 16) & 15][0], S.g, tc, S.mom[r]);
                }
                __syncthreads();
                if (threadIdx.x == 0) S.nruns = 0;
                for (int l = 0; l < ng; ++l) S.zb[l][threadIdx.x] = ZB_EMPTY;
                for (int j = threadIdx.x; j < n; j += NT) {        // gradients, one thread per bin face
                    for (int l = 0; l < ng; ++l) {
                        const int r = l * n + j;
                        if (__float_as_int(S.mom[r][9]) == 0) continue;
                        float dv[6], dc[9];
                        const SpanRec &R = S.rec[r];
                        face_grad(R, S.mom[r], t.fcol, dv, dc);
                        const float tau = S.taus[l];
                        if (j == (int)threadIdx.x) {   // the slot's persistent accumulator
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
                            flush(t, im, ch.s, R.fid, a0, a1, dc, dC);
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
                if (threadIdx.x == 0) S.taus[0] = tau;
                int base = 0, fpos = 0;
                while (true) {   // pass 1: the sub-frame's z-buffer over all batches
                    const int nb = next_batch(bc, t.F, tau, tc, t.W, t.H, SP_SREC_B, base, fpos, S.sid, S.wsum);
                    if (nb == 0) break;
                    __syncthreads();
                    stage_runs<false>(bc, nb, base, S.taus, 1, tc, t.W, t.H, t.F, S.sid, S.rec, S.runs, &S.nruns, wc);
                    __syncthreads();
                    walk_runs(S.rec, S.runs, S.nruns, tc, &S.zb[0][0], S.win);
                    __syncthreads();
                    if (threadIdx.x == 0) S.nruns = 0;
                    base += nb;
                }
                base = 0;
                fpos = 0;
                while (true) {   // pass 2: re-stage each batch, moments and gradients of its records
                    const int nb = next_batch(bc, t.F, tau, tc, t.W, t.H, SP_SREC_B, base, fpos, S.sid, S.wsum);
                    if (nb == 0) break;
                    __syncthreads();
                    stage_runs<false>(bc, nb, base, S.taus, 1, tc, t.W, t.H, t.F, S.sid, S.rec, S.runs, &S.nruns, wc);
                    __syncthreads();
                    if (threadIdx.x == 0) S.nruns = 0;
                    for (int j = threadIdx.x; j < nb; j += NT) {
                        const SpanRec &R = S.rec[j];
                        if (R.box < 0) continue;
                        if (rec_moments(R, S.runs, true, &S.zb[0][0], S.g, tc, S.mom[j]) == 0) continue;
                        float dv[6], dc[9], a0[6], a1[6];
                        face_grad(R, S.mom[j], t.fcol, dv, dc);
#pragma unroll
                        for (int i = 0; i < 6; ++i) { a0[i] = (1.f - tau) * dv[i]; a1[i] = tau * dv[i]; }
                        flush(t, im, ch.s, R.fid, a0, a1, dc, dC);
                    }
                    base += nb;
                    __syncthreads();
                }
                S.zb[0][threadIdx.x] = ZB_EMPTY;
                __syncthreads();
            }
        }
    }
}

template <bool CENSUS>
static cudaError_t launch_fwd_span(const Tables &t, float *out, int *ids, int ids_k, unsigned long long *census,
                                   cudaStream_t st)
{
    dim3 grid(t.T, t.B, t.splits);
    const int smem = (int)sizeof(SpFwdSmem);
    cudaError_t e = cudaFuncSetAttribute(k4s_raster_fwd<CENSUS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    k4s_raster_fwd<CENSUS><<<grid, NT, smem, st>>>(t, out, ids, ids_k, census);
    return cudaGetLastError();
}

cudaError_t launch_raster_fwd(const Tables &t, float *out, int *ids, int ids_k, unsigned long long *census,
                              cudaStream_t st)
{
    if (t.solver != 0 || t.legacy) return launch_raster_fwd_legacy(t, out, ids, ids_k, census, st);
    if (t.B == 0 || t.T == 0) return cudaSuccess;
    return census ? launch_fwd_span<true>(t, out, ids, ids_k, census, st)
                  : launch_fwd_span<false>(t, out, ids, ids_k, nullptr, st);
}

cudaError_t launch_raster_bwd(const Tables &t, const float *grad, float *dC, cudaStream_t st)
{
    if (t.solver != 0 || t.legacy) return launch_raster_bwd_legacy(t, grad, dC, st);
    if (t.B == 0 || t.T == 0 || t.F == 0) return cudaSuccess;
    dim3 grid(t.T, t.B, t.splits);
    const int smem = (int)sizeof(SpBwdSmem);
    cudaError_t e = cudaFuncSetAttribute(k6s_raster_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    k6s_raster_bwd<<<grid, NT, smem, st>>>(t, grad, dC);
    return cudaGetLastError();
}

}  // namespace br
