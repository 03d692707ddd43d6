// k_gather.cu -- K6 fused raster-backward from the bounded visibility cache ("visibility gather").
//
// Runs when K4 left the winning bin slot of every (pixel, sub-frame) of a chunk's bin in the
// workspace (BLUR_CACHE_VISIBILITY, bins of at most VIS_MAXN faces).  The
// gradient of the hard path (Q11: winner and coverage frozen) of a (face, sub-frame)
// record is the closed form of face_grad (raster_common.cuh) applied to nine moments of the pixels the
// face won, m = sum g (1, u, v) with g = dL/dI / N (Eq.9; dw/dv_i = -w_i dw/dp).
//
// One CTA = one 16x16 tile of one image (grid tiles x images x splits, like K4).  The CTA's chunk table
// is staged in shared memory once; its cached chunks are taken in super-groups of up to SG_T
// sub-frames and SG_SLOTS bin slots (several short chunks of a fast rotation share one group), so a
// group costs one HBM round trip for its winner words and one L2 round trip for its won records
// however its sub-frames are chunked:
//   load     thread = (sub-frame, 8-pixel row segment): the winner slots (16 B, coalesced) go to shared
//            memory; each run of equal winners sets its bit in the slot's 16-bit won mask (atomicOr).
//   list     thread = 4 consecutive group slots: a block scan of the won masks' popcounts lays out the
//            group's won pairs slot-major (pair index = slot base + rank of the sub-frame in the mask).
//   moments  thread = (sub-frame, segment): a run of equal winners takes its sums of q = round(g 2^e) and
//            q (x - 8) as two lookups in per-row prefix sums built once per CTA (q (8 - y) = dy x the first),
//            and adds them to its pair with native 32-bit shared atomics (integer sums: exact and
//            order-independent, deterministic, identical to summing the pixels; 2^e per tile with max |q| <
//            2^19, as k6_raster_bwd_fx).  (Summing the run's pixels one by one instead: C4 K6 3.36 ms vs 2.90.)
//   pairs    thread = won pair (face f at sub-frame tau): the face's segment record is evaluated at tau
//            (Eq.8 numerators and denominator by Horner, "computed only once" per segment) and
//            face_grad turns the moments into dL/dv (screen space) and dL/dc of the pair.
//   flush    thread = group slot: its pairs' gradients summed in sub-frame order, split (1 - tau, tau)
//            onto the segment's two keyframes (Eq.5-6); one vector RED per (vertex, keyframe) and three
//            REDs per vertex colour.
// Pairs beyond SG_PCAP are taken in further batches (moments, pairs, flush).  Chunks K4 wrote no
// winners for (longer bins, overflowed bins) are left to k6_raster_bwd_fx: the CTA raises its
// (image, tile) in Tables::vg_list, and k6_raster_bwd_fx runs only the listed tiles, skipping the chunks taken here.
#include <cstdio>

#include "internal.cuh"
#include "raster_common.cuh"
#include "../../include/blurrast.h"

namespace br {

#ifndef BR_SG_PCAP
#define BR_SG_PCAP 224
#endif
#ifndef BR_VG_SPLITS
#define BR_VG_SPLITS 1     // CTAs per (image, tile) (chunks dealt round-robin)
#endif
static_assert(BR_VG_SPLITS == 1, "the leftover list names whole (image, tile)s: one CTA must see all their chunks");
#ifndef BR_VG_PREFETCH
#define BR_VG_PREFETCH 0   // 1: L1 prefetch of the won faces' records in the list phase (C4 K6 +1%, C3 -2%)
#endif
#ifndef BR_VIS_STREAM
#define BR_VIS_STREAM 1   // streaming (evict-first) reads of the visibility cache (k_raster.cu: C4 step -0.4%)
#endif
#ifndef BR_VG_PREFIX
#define BR_VG_PREFIX 1     // 1: per-row prefix sums of the fixed-point pixel gradients; a run's moments are two lookups
#endif
#ifndef BR_VG_MINB
#define BR_VG_MINB 5
#endif
constexpr int SG_T = 16;                 // sub-frames per super-group (16-bit won masks)
constexpr int SG_SLOTS = 4 * NT;         // bin slots per super-group (4 per thread in the list phase)
constexpr int SG_PCAP = BR_SG_PCAP;      // won pairs per batch (moments + gradients in shared memory)
constexpr int SG_CMAX = 64;              // chunk-table window staged in shared memory
constexpr int SG_SEG = TW * TH / 8;      // 8-pixel row segments per tile
static_assert(VIS_MAXN <= SG_SLOTS, "a cached bin must fit a super-group");
static_assert(SG_T * SG_SEG == 2 * NT, "two (sub-frame, segment) items per thread");

struct __align__(16) VgSmem {
#if BR_VG_PREFIX
    int2 pq[TH][TW + 1][3];              // per row, prefix sums over x < k of q (rgb) and q (x - 8) (rgb), packed
                                         // (q.x, q.y) (q.z, u.x) (u.y, u.z): a run's moments are two lookups
#else
    int4 qg[TW * TH];                    // dL/dI / N of the tile (rgb) in fixed point, q = round(g 2^e)
#endif
    uint4 vis[SG_T][SG_SEG];             // winner slot per (group sub-frame, pixel), 0xFFFF none
    uint32_t wmask[SG_SLOTS / 2];        // won masks being built, two 16-bit slots per word
    uint32_t sbm[SG_SLOTS];              // per group slot: first pair index << 16 | won mask (bit l: won at sub-frame l)
    int imom[SG_PCAP][9];                // fixed-point moments M0 (rgb), Mu (rgb), Mv (rgb) per pair
    float contrib[SG_PCAP][15];          // per pair: dv (6, screen space), dc (9)
    int plist[SG_PCAP];                  // pairs of the batch: group slot | l << 10 | face id << 14 (-1 << 14: bad id)
    // chunk-table window of this CTA (chunks c_begin + z + i * splits)
    int ci_n[SG_CMAX], ci_k0[SG_CMAX], ci_ng[SG_CMAX], ci_s[SG_CMAX];
    long long ci_o[SG_CMAX];
    // group tables
    int t_k[SG_T];                       // image-local sub-frame index of group sub-frame l
    int t_soff[SG_T];                    // group slot of bin slot 0 of l's chunk
    int t_n[SG_T];                       // bin length of l's chunk
    float t_tau[SG_T];
    int t_seg[SG_T];                     // segment of l's chunk
    long long t_o[SG_T];                 // bin offset of l's chunk
    int wsum[NWARP];
    int left;                            // this CTA met chunks it does not take
};

struct PairRec {   // face_grad's view of a (face, sub-frame) record
    float a[3], b[3], g[3];
    float invD;
    int fid;
};

__device__ __forceinline__ uint16_t u4_get(const uint4 &w, int k)
{
    const unsigned x = k < 2 ? w.x : k < 4 ? w.y : k < 6 ? w.z : w.w;
    return (uint16_t)((k & 1) ? x >> 16 : x & 0xFFFFu);
}

// the face id of group slot gs (won at group sub-frame l0), -1 if out of range (never expected)
__device__ __forceinline__ int slot_face(const Tables &t, const VgSmem &S, int gs, int l0)
{
    const int f = __ldg(t.entries + S.t_o[l0] + (gs - S.t_soff[l0]));
    if ((unsigned)f >= (unsigned)t.F) {
        atomicOr(t.status, BLUR_ST_EINTERNAL);
        return -1;
    }
    return f;
}

// write the batch's pair codes (pairs [pb, pb + np)) of this thread's four group slots
__device__ __forceinline__ void write_plist(const Tables &t, VgSmem &S, int pb, int np)
{
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int gs = 4 * threadIdx.x + q;
        const uint32_t w = S.sbm[gs];
        unsigned mk = w & 0xFFFFu;
        if (!mk) continue;
        int i = (int)(w >> 16) - pb;
        if (i >= np || i + __popc(mk) <= 0) continue;
        const int f = slot_face(t, S, gs, __ffs(mk) - 1);
        for (; mk; mk &= mk - 1, ++i)
            if ((unsigned)i < (unsigned)np) S.plist[i] = gs | ((__ffs(mk) - 1) << 10) | (f << 14);
    }
}

__global__ void __launch_bounds__(NT, BR_VG_MINB) k6v_raster_bwd(Tables t, const float *__restrict__ grad,
                                                                float *__restrict__ dC)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    VgSmem &S = *reinterpret_cast<VgSmem *>(smem_raw);
    const int b = blockIdx.y, tile = blockIdx.x, tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    const ImgInfo &im = t.imgs[b];
    const int N = im.N, sched_off = im.sched_off;
    const int vsp = gridDim.z;   // CTAs per (image, tile), taking every vsp-th chunk
    const int cfirst = im.chunk_begin + (int)blockIdx.z;
    const int nc = cfirst < im.chunk_end ? (im.chunk_end - cfirst + vsp - 1) / vsp : 0;
    TileCtx tc;
    tile_ctx(t, tile, tc);
    {   // the tile's pixel gradients in fixed point: scale 2^e with max |g| 2^e < 2^19
        const int lx = tid & (TW - 1), ly = tid >> 4;
        float4 g = make_float4(0.f, 0.f, 0.f, 0.f);
        if (tc.px0 + lx < t.W && tc.py0 + ly < t.H) {
            g = __ldg(reinterpret_cast<const float4 *>(grad) + ((size_t)b * t.H + tc.py0 + ly) * t.W + tc.px0 + lx);
            const float inv = 1.0f / (float)N;   // dI/dI_k = 1/N (uniform mean)
            g.x *= inv; g.y *= inv; g.z *= inv;
        }
        float gm = fmaxf(fmaxf(fabsf(g.x), fabsf(g.y)), fabsf(g.z));
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) gm = fmaxf(gm, __shfl_xor_sync(0xffffffffu, gm, d));
        if (lane == 0) S.wsum[warp] = __float_as_int(gm);
        for (int i = tid; i < SG_SLOTS / 2; i += NT) S.wmask[i] = 0u;
        for (int i = tid; i < SG_PCAP * 9; i += NT) (&S.imom[0][0])[i] = 0;
        if (tid == 0) S.left = 0;
        __syncthreads();
        gm = 0.f;
#pragma unroll
        for (int w = 0; w < NWARP; ++w) gm = fmaxf(gm, __int_as_float(S.wsum[w]));
        int ex = 0;
        if (gm > 0.f) frexpf(gm, &ex);
        ex = min(max(ex, -100), 100);
        const float scale = ldexpf(1.0f, 19 - ex);
#if BR_VG_PREFIX
        {   // inclusive scans of q and q (x - 8) along the row (16 lanes of a half warp), exact in 32-bit integers
            int v[6];
            v[0] = __float2int_rn(g.x * scale); v[1] = __float2int_rn(g.y * scale); v[2] = __float2int_rn(g.z * scale);
            const int dx = lx - TW / 2;
            v[3] = v[0] * dx; v[4] = v[1] * dx; v[5] = v[2] * dx;
#pragma unroll
            for (int d = 1; d < TW; d <<= 1)
#pragma unroll
                for (int q = 0; q < 6; ++q) {
                    const int y = __shfl_up_sync(0xffffffffu, v[q], d, TW);
                    if (lx >= d) v[q] += y;
                }
            S.pq[ly][lx + 1][0] = make_int2(v[0], v[1]);
            S.pq[ly][lx + 1][1] = make_int2(v[2], v[3]);
            S.pq[ly][lx + 1][2] = make_int2(v[4], v[5]);
            if (lx == 0) {
                S.pq[ly][0][0] = make_int2(0, 0); S.pq[ly][0][1] = make_int2(0, 0); S.pq[ly][0][2] = make_int2(0, 0);
            }
        }
#else
        S.qg[tid] = make_int4(__float2int_rn(g.x * scale), __float2int_rn(g.y * scale), __float2int_rn(g.z * scale), 0);
#endif
    }
    float inv_scale;
    {
        float gm = 0.f;
#pragma unroll
        for (int w = 0; w < NWARP; ++w) gm = fmaxf(gm, __int_as_float(S.wsum[w]));
        int ex = 0;
        if (gm > 0.f) frexpf(gm, &ex);
        ex = min(max(ex, -100), 100);
        inv_scale = ldexpf(1.0f, ex - 19);
    }

    int ci = 0, w0 = -SG_CMAX;   // next chunk (CTA-local index) and the staged window [w0, w0 + SG_CMAX)
    while (true) {
        // ---- the next super-group: consecutive cached chunks of this CTA (uniform over the block)
        __syncthreads();   // the previous group has finished with the tables (and the window)
        if (ci >= w0 + SG_CMAX && ci < nc) {   // stage the next window of the chunk table
            w0 = ci;
            if (tid < SG_CMAX && w0 + tid < nc) {
                const int c = cfirst + (w0 + tid) * vsp;
                const Chunk ch = t.chunks[c];
                const size_t bi = (size_t)c * t.T + tile;
                const long long o = t.off[bi];
                const int n = (int)(t.off[bi + 1] - o);
                const bool cached = n > 0 && n <= VIS_MAXN && o + n <= t.cap;   // the bins K4 wrote winners for
                if (n > 0 && !cached) S.left = 1;
                S.ci_n[tid] = cached ? n : 0;
                S.ci_k0[tid] = ch.k0;
                S.ci_ng[tid] = ch.k1 - ch.k0;
                S.ci_s[tid] = ch.s;
                S.ci_o[tid] = o;
            }
            __syncthreads();
        }
        int L = 0, nsl = 0;
        while (ci < nc && ci < w0 + SG_CMAX) {
            const int wi = ci - w0;
            const int n = S.ci_n[wi];
            if (n == 0) { ++ci; continue; }
            const int ng = S.ci_ng[wi];
            if (L + ng > SG_T || nsl + n > SG_SLOTS) break;
            if (tid < ng) {
                const int l = L + tid;
                S.t_k[l] = S.ci_k0[wi] + tid;
                S.t_soff[l] = nsl;
                S.t_n[l] = n;
                S.t_tau[l] = t.sched_tau[sched_off + S.ci_k0[wi] + tid];
                S.t_seg[l] = S.ci_s[wi];
                S.t_o[l] = S.ci_o[wi];
            }
            L += ng;
            nsl += n;
            ++ci;
        }
        if (L == 0) {
            if (ci < nc) continue;   // window exhausted by uncached chunks: stage the next one
            break;
        }
        __syncthreads();
        // ---- load: winners of the group's sub-frames -> shared memory, won masks
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int it = tid + h * NT, l = it / SG_SEG, sg = it % SG_SEG;
            if (l >= L) continue;
            const int row = sg >> 1, x0 = (sg & 1) * 8;
#if BR_VIS_STREAM
            uint4 w = __ldcs(reinterpret_cast<const uint4 *>(t.vis + ((size_t)(im.cov_off + S.t_k[l]) * t.T + tile) * (TW * TH)) + sg);
#else
            uint4 w = reinterpret_cast<const uint4 *>(t.vis + ((size_t)(im.cov_off + S.t_k[l]) * t.T + tile) * (TW * TH))[sg];
#endif
            const int n = S.t_n[l], soff = S.t_soff[l];
            const bool rowin = tc.py0 + row < t.H;
            unsigned ow[4] = {0u, 0u, 0u, 0u};
            int prev = -1;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                int e = u4_get(w, k);
                if (!rowin || tc.px0 + x0 + k >= t.W) e = 0xFFFF;
                if (e != 0xFFFF && e >= n) {   // never expected: K4 writes slots of this bin
                    atomicOr(t.status, BLUR_ST_EINTERNAL);
                    e = 0xFFFF;
                }
                ow[k >> 1] |= (unsigned)e << ((k & 1) * 16);
                if (e != 0xFFFF && e != prev) {
                    const int gs = soff + e;
                    atomicOr(&S.wmask[gs >> 1], 1u << (l + 16 * (gs & 1)));
                }
                prev = e;
            }
            S.vis[l][sg] = make_uint4(ow[0], ow[1], ow[2], ow[3]);
        }
        __syncthreads();
        // ---- list: masks, slot bases (block scan over the group's slots, 4 per thread)
        int total;
        {
            const uint32_t w0m = S.wmask[2 * tid], w1m = S.wmask[2 * tid + 1];
            S.wmask[2 * tid] = 0u;
            S.wmask[2 * tid + 1] = 0u;
            const unsigned mk[4] = {w0m & 0xFFFFu, w0m >> 16, w1m & 0xFFFFu, w1m >> 16};
            int cnt = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) cnt += __popc(mk[q]);
            int x = cnt;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, x, d);
                if (lane >= d) x += y;
            }
            if (lane == 31) S.wsum[warp] = x;
            __syncthreads();
            int base = x - cnt;
            total = 0;
#pragma unroll
            for (int w = 0; w < NWARP; ++w) {
                const int s = S.wsum[w];
                base += w < warp ? s : 0;
                total += s;
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int gs = 4 * tid + q;
                S.sbm[gs] = ((uint32_t)base << 16) | mk[q];
                if (mk[q] && base < SG_PCAP) {
                    // the slot's chunk: that of its first won sub-frame
                    const int l0 = __ffs(mk[q]) - 1;
                    const int f = slot_face(t, S, gs, l0);
#if BR_VG_PREFETCH
                    if (f >= 0) {   // the pair phase reads the face's segment record and colours: start them now
                        const float4 *rr = t.rec + ((size_t)(im.rec_off + (long long)S.t_seg[l0] * t.F) + f) * REC_F4;
                        asm volatile("prefetch.global.L1 [%0];" ::"l"(rr));
                        asm volatile("prefetch.global.L1 [%0];" ::"l"(rr + 6));
                        asm volatile("prefetch.global.L1 [%0];" ::"l"(t.fcol + 3 * (size_t)f));
                    }
#endif
                    int i = base;
                    for (unsigned m = mk[q]; m; m &= m - 1, ++i)
                        if (i < SG_PCAP) S.plist[i] = gs | ((__ffs(m) - 1) << 10) | (f << 14);
                }
                base += __popc(mk[q]);
            }
        }
        __syncthreads();
        // ---- batches of SG_PCAP pairs: moments, pair gradients, flush
        for (int pb = 0; pb < total; pb += SG_PCAP) {
            const int np = min(SG_PCAP, total - pb);
            if (pb > 0) {
                write_plist(t, S, pb, np);
                __syncthreads();
            }
            // moments (imom is zero on entry: cleared at start and by every pair that read it)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int it = tid + h * NT, l = it / SG_SEG, sg = it % SG_SEG;
                if (l >= L) continue;
                const uint4 w = S.vis[l][sg];
                const int soff = S.t_soff[l], row = sg >> 1, x0 = (sg & 1) * 8;
                const int dy = TH / 2 - row;
                const unsigned low = (1u << l) - 1u;   // (< 2^15: selects mask bits only)
                int cur = -1, prev = -1;
                int m0 = 0, m1 = 0, m2 = 0, u0 = 0, u1 = 0, u2 = 0;
#if BR_VG_PREFIX
                int ka = 0;   // first pixel of the current run
#endif
#pragma unroll
                for (int k = 0; k <= 8; ++k) {
                    const int e = k < 8 ? (int)u4_get(w, k) : 0xFFFF;
                    if (e != prev) {   // run boundary: add the finished run, start the next
#if BR_VG_PREFIX
                        if (cur >= 0) {   // the run [ka, k) of this segment: prefix differences
                            const int2 *pa = S.pq[row][x0 + ka], *pb = S.pq[row][x0 + k];
                            const int2 a0 = pa[0], a1 = pa[1], a2 = pa[2], b0 = pb[0], b1 = pb[1], b2 = pb[2];
                            m0 = b0.x - a0.x; m1 = b0.y - a0.y; m2 = b1.x - a1.x;
                            u0 = b1.y - a1.y; u1 = b2.x - a2.x; u2 = b2.y - a2.y;
                        }
                        ka = k;
#endif
                        if (cur >= 0) {
                            int *m = S.imom[cur];
                            atomicAdd(m + 0, m0); atomicAdd(m + 1, m1); atomicAdd(m + 2, m2);
                            atomicAdd(m + 3, u0); atomicAdd(m + 4, u1); atomicAdd(m + 5, u2);
                            atomicAdd(m + 6, m0 * dy); atomicAdd(m + 7, m1 * dy); atomicAdd(m + 8, m2 * dy);   // dy is constant over the row
                        }
                        cur = -1;
                        if (e != 0xFFFF) {
                            const int gs = soff + e;
                            const uint32_t w = S.sbm[gs];
                            const int pi = (int)(w >> 16) + __popc(w & low) - pb;
                            cur = (unsigned)pi < (unsigned)np ? pi : -1;
                        }
                        m0 = m1 = m2 = u0 = u1 = u2 = 0;
                        prev = e;
                    }
#if !BR_VG_PREFIX
                    if (k < 8 && cur >= 0) {
                        const int4 q = S.qg[row * TW + x0 + k];
                        const int dx = x0 + k - TW / 2;
                        m0 += q.x; m1 += q.y; m2 += q.z;
                        u0 += q.x * dx; u1 += q.y * dx; u2 += q.z * dx;
                    }
#endif
                }
            }
            __syncthreads();
            // pairs: thread per pair
            for (int i = tid; i < np; i += NT) {
                const int code = S.plist[i];
                const int l = (code >> 10) & 0xF, fj = code >> 14;
                int *mi = S.imom[i];
                float m[9];
#pragma unroll
                for (int q = 0; q < 3; ++q) {
                    m[q] = (float)mi[q] * inv_scale;
                    m[3 + q] = (float)mi[3 + q] * inv_scale * tc.sx;
                    m[6 + q] = (float)mi[6 + q] * inv_scale * tc.sy;
                }
#pragma unroll
                for (int q = 0; q < 9; ++q) mi[q] = 0;
                float dv[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f}, dc[9] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
                if (fj >= 0) {
                    const float tau = S.t_tau[l];
                    const float4 *rr = t.rec + ((size_t)(im.rec_off + (long long)S.t_seg[l] * t.F) + fj) * REC_F4;
                    const float4 q6 = __ldg(rr + 6);
                    const float D = __fmaf_rn(tau, __fmaf_rn(tau, q6.x, q6.y), q6.z);   // det F(tau) (Eq.8)
                    // the record at tau for this tile, as K4's stage: sign-normalised, tile-centred
                    PairRec pr;
                    const float sgn = D < 0.f ? -1.f : 1.f;
                    pr.invD = 1.0f / fabsf(D);
                    pr.fid = fj;
#pragma unroll
                    for (int e = 0; e < 3; ++e) {
                        const float4 qa = __ldg(rr + 2 * e), qb = __ldg(rr + 2 * e + 1);   // ox oy a0 a1 | b0 b1 dax day
                        float al, be, gp;
                        rec_edge_at(qa, qb, tau, tc.uc, tc.vc, al, be, gp);
                        pr.a[e] = al * sgn;
                        pr.b[e] = be * sgn;
                        pr.g[e] = gp * sgn;
                    }
                    face_grad(pr, m, t.fcol, dv, dc);
                }
                float *cb = S.contrib[i];
#pragma unroll
                for (int e = 0; e < 6; ++e) cb[e] = dv[e];
#pragma unroll
                for (int e = 0; e < 9; ++e) cb[6 + e] = dc[e];
            }
            __syncthreads();
            // flush: thread per group slot, its pairs of this batch in sub-frame order
            for (int gs = tid; gs < nsl; gs += NT) {
                const uint32_t w = S.sbm[gs];
                const unsigned mk = w & 0xFFFFu;
                if (!mk) continue;
                const int base = (int)(w >> 16);
                if (base >= pb + np || base + __popc(mk) <= pb) continue;
                FaceAcc acc;
                acc_zero(acc);
                const int l0 = __ffs(mk) - 1;
                int i = base;
                for (unsigned mm = mk; mm; mm &= mm - 1, ++i) {
                    if (i < pb || i >= pb + np) continue;
                    const float *cb = S.contrib[i - pb];
                    const float tau = S.t_tau[__ffs(mm) - 1];
#pragma unroll
                    for (int e = 0; e < 6; ++e) {
                        acc.k0[e] = __fmaf_rn(1.f - tau, cb[e], acc.k0[e]);
                        acc.k1[e] = __fmaf_rn(tau, cb[e], acc.k1[e]);
                    }
#pragma unroll
                    for (int e = 0; e < 9; ++e) acc.c[e] += cb[6 + e];
                }
                const int fj = S.plist[max(base, pb) - pb] >> 14;
                if (fj >= 0) flush(t, im, S.t_seg[l0], fj, acc.k0, acc.k1, acc.c, dC);
            }
            if (pb + np < total) __syncthreads();   // the next batch reuses plist / imom / contrib
        }
    }
    if (tid == 0 && S.left)   // list the (image, tile) for k6_raster_bwd_fx (count zeroed by K1 and by K7 of the previous backward)
        t.vg_list[atomicAdd(t.vg_count, 1)] = blockIdx.y * t.T + blockIdx.x;
}

cudaError_t launch_vis_gather(const Tables &t, const float *grad, float *dC, cudaStream_t st)
{
    dim3 grid(t.T, t.B, BR_VG_SPLITS);
    const int smem = (int)sizeof(VgSmem);

    cudaError_t e = cudaFuncSetAttribute(k6v_raster_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    k6v_raster_bwd<<<grid, NT, smem, st>>>(t, grad, dC);
    return cudaGetLastError();
}

}  // namespace br
