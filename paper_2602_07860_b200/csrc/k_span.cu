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

struct __align__(16) SpanRec {   // a (face, sub-frame) record for this tile, 80 B
    float b[3], g[3];            // sign-normalised edge functions e_i = a_i ul + b_i vl + g_i (tile-local)
    float k[3];                  // -1 / (a_i sx) (0 where a_i = 0): edge i bounds a row at x = TW/2 + k_i R_i(v)
    int box;                     // x0 | x1 << 4 | y0 << 8 | y1 << 12 (tile-local pixel box) | l << 16 (sub-frame
                                 // layer); -1: no record
    float az, bz, cz;            // depth plane z = fma(az, ul, fma(bz, vl, cz)) (Q6)
    unsigned tag;                // z-buffer key low word: fid << 10 | slot j
    float invD;                  // 1 / |det F(tau)|
    int fid;
    float a[3];
    float pad;
};
static_assert(SP_GMAX <= 16, "layer field of SpanRec::box is 4 bits");

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
// Every edge function e_i(x) = fma(A_i, ul(x), R_i) of the row (R_i = fma(B_i, vl, G_i)) is monotone in x
// (a correctly rounded fma of an increasing ul(x)), so the covered pixels form one interval, bounded below
// by the edges with A_i > 0 (k_i < 0) and above by those with A_i < 0 (k_i > 0); an edge's boundary is
// x* = TW/2 + k_i R_i, k_i = -1 / (A_i sx).  Evaluated from the row's exact R_i it carries an error of a few
// ulp of |x* - TW/2|, i.e. < 1e-5 px wherever the boundary is inside the tile (edges with A_i = 0 restrict
// the record's rows instead, span_setup).  A range end within SPAN_DLT of a boundary is re-tested with the
// per-pixel arithmetic itself, scanning inward, so the result is exactly the set of pixels of the row
// that pass cov_at.  Returns the number of exact tests taken (census).
__device__ __forceinline__ int row_range(const SpanRec &Rec, int y, int x0, int x1, const TileCtx &tc, int &lo,
                                         int &hi)
{
    const float vl = (float)(TH / 2 - y) * tc.sy;
    float L = -100.5f, U = 116.5f;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const float R = __fmaf_rn(Rec.b[i], vl, Rec.g[i]);
        const float t = fmaf(R, Rec.k[i], (float)(TW / 2));
        L = Rec.k[i] < 0.f ? fmaxf(L, t) : L;
        U = Rec.k[i] > 0.f ? fminf(U, t) : U;
    }
    L = fminf(L, 116.5f);
    U = fmaxf(U, -100.5f);
    const float cl = ceilf(L - SPAN_DLT), ch = floorf(U + SPAN_DLT);
    lo = max((int)cl, x0);
    hi = min((int)ch, x1);
    int nt = 0;
    if (lo <= hi && (cl <= L + SPAN_DLT || ch >= U - SPAN_DLT)) {
        // a range end within SPAN_DLT of a boundary: move the ends inward with the exact test
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
    const float dzb = zb - za, dzc = zc - za;
    az = __fmaf_rn(A[1], dzb, A[2] * dzc) * invD;
    bz = __fmaf_rn(B[1], dzb, B[2] * dzc) * invD;
    cz = __fmaf_rn(__fmaf_rn(G[1], dzb, G[2] * dzc), invD, za);
}

// The row bounds of the record (see row_range): k_i = -1/(A_i sx), clamped to +-1e30 (finite even where
// A_i sx underflows; the boundary of an edge with A_i ~ 0 lies far off the tile unless R_i ~ 0, and then
// at TW/2, where it is), 0 for A_i = 0.  An edge with A_i = 0 has e_i = R_i on the whole row: rows with
// R_i < 0 are dropped from [y0, y1] (R_i is monotone in the row).  Returns false when no row is left.
__device__ __forceinline__ bool span_setup(const float A[3], const float B[3], const float G[3], const TileCtx &tc,
                                           int &y0, int &y1, float K[3])
{
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const float as = A[i] * tc.sx;
        K[i] = as != 0.f ? fminf(fmaxf(-__frcp_rn(as), -1e30f), 1e30f) : 0.f;
        if (A[i] == 0.f) {
            while (y0 <= y1 && __fmaf_rn(B[i], (float)(TH / 2 - y0) * tc.sy, G[i]) < 0.f) ++y0;
            while (y0 <= y1 && __fmaf_rn(B[i], (float)(TH / 2 - y1) * tc.sy, G[i]) < 0.f) --y1;
        }
    }
    return y0 <= y1;
}

__device__ __forceinline__ void store_rec(SpanRec &o, const float A[3], const float B[3], const float G[3], float invD,
                                          int fid, int box, const float K[3], float az, float bz, float cz,
                                          unsigned tag)
{
    float4 *q = reinterpret_cast<float4 *>(&o);
    q[0] = make_float4(B[0], B[1], B[2], G[0]);
    q[1] = make_float4(G[1], G[2], K[0], K[1]);
    q[2] = make_float4(K[2], __int_as_float(box), az, bz);
    q[3] = make_float4(cz, __uint_as_float(tag), invD, __int_as_float(fid));
    q[4] = make_float4(A[0], A[1], A[2], 0.f);
}

struct WalkCount {
    unsigned long long frag = 0, test = 0, rec = 0;
};

// Stage the bin faces [base, base+nb) (or sid[] on the fallback path) at the ng sub-frames taus[0..ng):
// one thread per (face j, sub-frame l) pair builds the record rec[l * nb + j] (edge functions, boundary
// lines, depth plane) and appends one unit (record << 4 | row) per row of its pixel box to units[]
// (one shared atomic per warp).  Pairs without coverage get box = -1.  Work is spread face-major, so
// lanes sharing a face load its (face, segment) record with broadcast loads.
template <bool CENSUS>
__device__ __forceinline__ void stage_units(const BinCtx &bc, int nb, int base, const float *taus, int ng,
                                            const TileCtx &tc, int W, int H, int F, const int *sid, SpanRec *rec,
                                            uint16_t *units, int *nunits, WalkCount &wc)
{
    const int lane = threadIdx.x & 31;
    const float inv_ng = 1.0f / (float)ng;
    const int npair = nb * ng;
    for (int p0 = 0; p0 < npair; p0 += NT) {   // block-uniform trip count: the warp scan below is convergent
        const int p = p0 + threadIdx.x;
        int rows = 0, y0 = 0, r = 0;
        if (p < npair) {
            const int j = div_small(p, inv_ng), l = p - j * ng;
            r = l * nb + j;
            SpanRec &out = rec[r];
            out.box = -1;
            const int f = bc.fb ? sid[j] : __ldg(bc.ent + base + j);
            if ((unsigned)f >= (unsigned)F) {     // never expected: bins hold valid face ids
                atomicOr(bc.status, BLUR_ST_EINTERNAL);
            } else {
                const float4 *rp = bc.rseg + (size_t)f * REC_F4;
                const float4 q6 = __ldg(rp + 6);
                const float tau = taus[l];
                const float D = __fmaf_rn(tau, __fmaf_rn(tau, q6.x, q6.y), q6.z);   // det F(tau), A8
                int x0 = 0, x1 = -1, y1 = -1;
                bool ok = __float_as_int(q6.w) >= 0 && fabsf(D) > EPS_D;          // skipped face; Q8
                if (ok) {
                    const float4 b0 = __ldg(rp + 7), b1 = __ldg(rp + 8);
                    ok = tile_pixels(box_lerp(tau, b0.x, b1.x), box_lerp(tau, b0.y, b1.y), box_lerp(tau, b0.z, b1.z),
                                     box_lerp(tau, b0.w, b1.w), W, H, tc, x0, x1, y0, y1);
                }
                if (ok) {
                    FaceRec fr;
                    load_rec(rp, fr);
                    float A[3], B[3], G[3], invD, az, bz, cz, K[3];
                    eval_tau(fr, tau, D, tc, A, B, G, invD, az, bz, cz);
                    if (span_setup(A, B, G, tc, y0, y1, K)) {
                        const int fid = __float_as_int(q6.w);
                        store_rec(out, A, B, G, invD, fid, x0 | (x1 << 4) | (y0 << 8) | (y1 << 12) | (l << 16), K, az,
                                  bz, cz, ((unsigned)fid << 10) | (unsigned)j);
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
        if (lane == 31 && tot > 0) b0 = atomicAdd(nunits, tot);
        b0 = __shfl_sync(0xffffffffu, b0, 31) + incl - rows;
        for (int k = 0; k < rows; ++k) units[b0 + k] = (uint16_t)((r << 4) | (y0 + k));
    }
}

// Walk the units[0..nu): one thread per (record, row) finds the row's exact covered range (row_range);
// the covered pixels of each warp's 32 units are then spread evenly over its lanes (rounds of 32 pixels:
// each lane finds the unit its pixel belongs to from the units' start positions in the round and takes
// the unit's data by shuffles), and every covered pixel offers its key (order(depth) << 32 | fid << 10 |
// slot j) to the z-buffer layer of the record's sub-frame (64-bit shared CAS min).  win: 32 ints per warp.
template <bool CENSUS>
__device__ __forceinline__ void walk_units(const SpanRec *rec, const uint16_t *units, int nu, const TileCtx &tc,
                                           unsigned long long *zb, int *wwin, WalkCount &wc)
{
    const int lane = threadIdx.x & 31;
    int *win = wwin + (threadIdx.x >> 5) * 32;
    for (int u0 = 0; u0 < nu; u0 += NT) {   // block-uniform trip count (the warp collectives are convergent)
        const int u = u0 + (int)threadIdx.x;
        int lo = 0, cnt = 0, zoff = 0;
        float az = 0.f, rz = 0.f;
        unsigned tag = 0;
        if (u < nu) {
            const unsigned e = units[u];
            const int r = (int)(e >> 4), y = (int)(e & 15u);
            const SpanRec &R = rec[r];
            const int box = R.box;
            int hi;
            const int nt = row_range(R, y, box & 15, (box >> 4) & 15, tc, lo, hi);
            cnt = hi >= lo ? hi - lo + 1 : 0;
            if (CENSUS) { wc.test += nt; wc.frag += cnt; }
            const float vl = (float)(TH / 2 - y) * tc.sy;
            az = R.az;
            rz = __fmaf_rn(R.bz, vl, R.cz);
            tag = R.tag;
            zoff = ((box >> 16) & 15) * (TW * TH) + y * TW;
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
            // units starting in this round mark their start position; the other pixels of the round belong
            // to the last unit started before it (the carried one)
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
    uint16_t units[SP_SREC_F * TH];   // (record, row) work items of the group: record << 4 | row
    int sid[SP_SREC_F];
    float taus[SP_GMAX];
    int wsum[NWARP];
    int nunits;
    int win[NWARP * 32];   // walk_units: per-warp owner windows
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
    if (threadIdx.x == 0) S.nunits = 0;
    WalkCount wc;
    unsigned long long nshade = 0, ngroup = 0, npairs = 0, nsub = 0;
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
                if (CENSUS) { ngroup++; npairs += n * ng; nsub += ng; }
                if (threadIdx.x < ng) S.taus[threadIdx.x] = t.sched_tau[sched_off + kg + threadIdx.x];
                __syncthreads();
                stage_units<CENSUS>(bc, n, 0, S.taus, ng, tc, t.W, t.H, t.F, S.sid, S.rec, S.units, &S.nunits, wc);
                __syncthreads();
                walk_units<CENSUS>(S.rec, S.units, S.nunits, tc, &S.zb[0][0], S.win, wc);
                __syncthreads();
                if (threadIdx.x == 0) S.nunits = 0;
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
                    stage_units<CENSUS>(bc, nb, base, S.taus, 1, tc, t.W, t.H, t.F, S.sid, S.rec, S.units, &S.nunits, wc);
                    __syncthreads();
                    walk_units<CENSUS>(S.rec, S.units, S.nunits, tc, &S.zb[0][0], S.win, wc);
                    __syncthreads();
                    if (threadIdx.x == 0) S.nunits = 0;
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
        if (threadIdx.x == 0) {   // grouped-path shape (diagnostics): groups, (face, sub-frame) pairs, sub-frames
            atomicAdd(census + 5, ngroup);
            atomicAdd(census + 6, npairs);
            atomicAdd(census + 7, nsub);
        }
    }
}

// ------------------------------------------------------------------ backward
//
// The z-buffer is rebuilt exactly as in the forward (stage_units + walk_units).  Then one thread per
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
    uint16_t units[SP_SREC_B * TH];
    float mom[SP_SREC_B][10];   // per record: the nine moments of its won pixels and their count
    float4 g[TW * TH];          // dL/dI / N of the tile
    int sid[SP_SREC_B];
    float taus[SP_GMAX_B];
    int wsum[NWARP];
    int nunits;
    int win[NWARP * 32];
};

// moments of the pixels record r won (key low word == tag, or with by_fid (batched path: slots repeat
// across batches) key low word >> 10 == fid) over its rows, into mo[0..9]; returns the count
__device__ __forceinline__ int rec_moments(const SpanRec &R, bool by_fid, const unsigned long long *zl,
                                           const float4 *g, const TileCtx &tc, float *mo)
{
    const int box = R.box;
    const int x0 = box & 15, x1 = (box >> 4) & 15, y0 = (box >> 8) & 15, y1 = (box >> 12) & 15;
    const unsigned tag = R.tag, fid = (unsigned)R.fid;
    float m[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) m[q] = 0.f;
    int cnt = 0;
    const unsigned *zw = reinterpret_cast<const unsigned *>(zl);
    for (int y = y0; y <= y1; ++y) {
        int lo, hi;
        row_range(R, y, x0, x1, tc, lo, hi);
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
    if (threadIdx.x == 0) S.nunits = 0;
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
                stage_units<false>(bc, n, 0, S.taus, ng, tc, t.W, t.H, t.F, S.sid, S.rec, S.units, &S.nunits, wc);
                __syncthreads();
                walk_units<false>(S.rec, S.units, S.nunits, tc, &S.zb[0][0], S.win, wc);
                __syncthreads();
                for (int r = threadIdx.x; r < n * ng; r += NT) {   // moments, one thread per record
                    const SpanRec &R = S.rec[r];
                    if (R.box < 0) { S.mom[r][9] = 0.f; continue; }
                    rec_moments(R, false, &S.zb[(R.box >> 16) & 15][0], S.g, tc, S.mom[r]);
                }
                __syncthreads();
                if (threadIdx.x == 0) S.nunits = 0;
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
                    stage_units<false>(bc, nb, base, S.taus, 1, tc, t.W, t.H, t.F, S.sid, S.rec, S.units, &S.nunits, wc);
                    __syncthreads();
                    walk_units<false>(S.rec, S.units, S.nunits, tc, &S.zb[0][0], S.win, wc);
                    __syncthreads();
                    if (threadIdx.x == 0) S.nunits = 0;
                    base += nb;
                }
                base = 0;
                fpos = 0;
                while (true) {   // pass 2: re-stage each batch, moments and gradients of its records
                    const int nb = next_batch(bc, t.F, tau, tc, t.W, t.H, SP_SREC_B, base, fpos, S.sid, S.wsum);
                    if (nb == 0) break;
                    __syncthreads();
                    stage_units<false>(bc, nb, base, S.taus, 1, tc, t.W, t.H, t.F, S.sid, S.rec, S.units, &S.nunits, wc);
                    __syncthreads();
                    if (threadIdx.x == 0) S.nunits = 0;
                    for (int j = threadIdx.x; j < nb; j += NT) {
                        const SpanRec &R = S.rec[j];
                        if (R.box < 0) continue;
                        if (rec_moments(R, true, &S.zb[0][0], S.g, tc, S.mom[j]) == 0) continue;
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
