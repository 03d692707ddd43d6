// k_raster.cu -- K4 fused raster-forward and K6 fused raster-backward.
//
// One CTA = one 16x16 pixel tile of one image; 8 warps, each owning an 8x4 footprint, one pixel
// per thread.  For every chunk of sub-frames the CTA reads the tile's bin (faces sorted by index).
// For every sub-frame tau of the chunk:
//   stage   each face of the bin evaluates its segment coefficients at tau (Eq.8 numerators and
//           denominator, Horner in tau -- "compute once, evaluate per sample") about the tile
//           centre, normalises the sign by det F(tau) and writes a 64 B record to shared memory,
//           with its per-tau pixel box (tile-level cull) -> sbox
//   vis     each warp culls the staged faces against its 8x4 footprint (lanes test 32 boxes at a
//           time, ballot) and every lane evaluates the three numerators at its pixel centre
//           (2 FMA each), tests coverage by sign (all w_i >= 0), and keeps the nearest face
//           (z-buffer in registers, strict <, faces in index order -> lower index wins ties, Q7)
//   shade   fwd: w_i = N_i / |D|, I = sum w_i c_i (Eq.9), accumulated in registers over all
//           sub-frames; the sub-frames never reach HBM.  Output (1/N) sum, written once.
//           bwd: the winner map goes to shared memory; each face thread walks its pixel box,
//           gathers dL/dI at the pixels it won and accumulates colour and screen-position
//           gradients in registers (aggregated over pixels and over the chunk's sub-frames), then
//           flushes them with one vector atomic per (vertex, keyframe).
// Bins that overflowed (or exceed SORTCAP) are regenerated exactly by scanning all faces in index
// order (slow path).  Faces of a bin above CAP are processed in several batches.
#include <cstdio>

#include "internal.cuh"
#include "../../include/blurrast.h"

namespace br {

constexpr uint32_t EMPTY_BOX = 0x001F001Fu;   // x0 = 31 > x1 = 0 -> never overlaps

struct TileCtx {
    float uc, vc;     // NDC of the tile's reference pixel centre (TW/2, TH/2)
    float sx, sy;     // 2/W, 2/H
    int px0, py0;     // tile origin (pixels)
    int lxmax, lymax; // last in-image local pixel
};

__device__ __forceinline__ float edge_eval(float a, float b, float g, float ul, float vl)
{
    return __fmaf_rn(a, ul, __fmaf_rn(b, vl, g));
}

__device__ __forceinline__ bool tile_pixels(float xmn, float xmx, float ymn, float ymx, int W, int H,
                                            const TileCtx &tc, int &x0, int &x1, int &y0, int &y1)
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

// Evaluate the (face, segment) record at tau for this tile -> TauRec + packed pixel box.
__device__ __forceinline__ void stage_one(const float4 *__restrict__ r, float tau, const TileCtx &tc,
                                          int W, int H, TauRec &out, uint32_t &box)
{
    box = EMPTY_BOX;
    const float4 q6 = __ldg(r + 6);
    const int fid = __float_as_int(q6.w);
    out.fid = fid;
    if (fid < 0) return;
    const float D = __fmaf_rn(tau, __fmaf_rn(tau, q6.x, q6.y), q6.z);   // a1 t^2 + a2 t + a3
    if (!(fabsf(D) > EPS_D)) return;                                    // Q8
    const float4 b0 = __ldg(r + 7), b1 = __ldg(r + 8);
    int x0, x1, y0, y1;
    if (!tile_pixels(box_lerp(tau, b0.x, b1.x), box_lerp(tau, b0.y, b1.y), box_lerp(tau, b0.z, b1.z),
                     box_lerp(tau, b0.w, b1.w), W, H, tc, x0, x1, y0, y1))
        return;
    const float sg = D < 0.f ? -1.f : 1.f;
    const float invD = 1.0f / fabsf(D);
    float A[3], B[3], G[3];
    float4 e[6];
#pragma unroll
    for (int q = 0; q < 6; ++q) e[q] = __ldg(r + q);
    const float *ef = reinterpret_cast<const float *>(e);
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
    // tile-level reject: the edge function's maximum over the tile's pixel centres
    const float ulmin = -(TW / 2) * tc.sx, ulmax = (TW / 2 - 1) * tc.sx;
    const float vlmin = -(TH / 2 - 1) * tc.sy, vlmax = (TH / 2) * tc.sy;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const float m = G[i] + (A[i] > 0.f ? A[i] * ulmax : A[i] * ulmin) + (B[i] > 0.f ? B[i] * vlmax : B[i] * vlmin);
        const float tol = 1e-6f * (fabsf(A[i]) * ulmax + fabsf(B[i]) * vlmax + fabsf(G[i])) + 1e-30f;
        if (m < -tol) return;
    }
    const float4 z0 = __ldg(r + 9), z1 = __ldg(r + 10);
    const float za = __fmaf_rn(tau, z1.x - z0.x, z0.x);
    const float zb = __fmaf_rn(tau, z1.y - z0.y, z0.y);
    const float zc = __fmaf_rn(tau, z1.z - z0.z, z0.z);
    out.a[0] = A[0]; out.a[1] = A[1]; out.a[2] = A[2];
    out.b[0] = B[0]; out.b[1] = B[1]; out.b[2] = B[2];
    out.g[0] = G[0]; out.g[1] = G[1]; out.g[2] = G[2];
    // depth interpolated with the screen-space weights (Q6): z(p) = sum_i w_i(p) z_i, written as
    // z0 + w1 (z1 - z0) + w2 (z2 - z0).  Same plane when sum_i w_i = 1; in fp32 the weights of a
    // sliver face sum to 1 +- 1e-4, and this form keeps that error off the absolute depth.
    const float dzb = zb - za, dzc = zc - za;
    out.az = __fmaf_rn(A[1], dzb, A[2] * dzc) * invD;
    out.bz = __fmaf_rn(B[1], dzb, B[2] * dzc) * invD;
    out.cz = __fmaf_rn(__fmaf_rn(G[1], dzb, G[2] * dzc), invD, za);
    out.invD = invD;
    box = (uint32_t)x0 | ((uint32_t)x1 << 8) | ((uint32_t)y0 << 16) | ((uint32_t)y1 << 24);
}

// Fallback batch builder: faces whose per-tau box overlaps the tile, in index order, from fpos on.
// Block-uniform.  Returns the batch size (0 when all faces are consumed).
__device__ int fallback_fill(const float4 *__restrict__ rseg, int F, float tau, const TileCtx &tc, int W,
                             int H, int &fpos, int *sid, int *swsum)
{
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int nb = 0;
    while (fpos < F) {
        const int f = fpos + tid;
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
        if (lane == 0) swsum[warp] = __popc(m);
        __syncthreads();
        int pre = 0, tot = 0;
#pragma unroll
        for (int w = 0; w < NT / 32; ++w) {
            const int c = swsum[w];
            pre += w < warp ? c : 0;
            tot += c;
        }
        __syncthreads();
        if (nb + tot > CAP) break;                       // uniform: batch full
        if (hit) sid[nb + pre + __popc(m & ((1u << lane) - 1u))] = f;
        nb += tot;
        fpos += NT;
    }
    __syncthreads();   // sid[] complete before the batch is staged
    return nb;
}

struct BinCtx {
    int *status;
    const float4 *rseg;   // records of (image, segment)
    const int *ent;       // sorted bin entries (normal path)
    int n;                // bin length
    bool fb;              // fallback path
};

// Batch iteration shared by the passes: returns nb (0 = done).  Normal path: contiguous slices of
// the sorted bin.  Fallback: regenerated by scanning faces.
__device__ __forceinline__ int next_batch(const BinCtx &bc, int F, float tau, const TileCtx &tc, int W, int H,
                                          int base, int &fpos, int *sid, int *swsum)
{
    if (!bc.fb) return base < bc.n ? min(CAP, bc.n - base) : 0;
    return fallback_fill(bc.rseg, F, tau, tc, W, H, fpos, sid, swsum);
}

__device__ __forceinline__ void stage_batch(const BinCtx &bc, int nb, int base, float tau, const TileCtx &tc,
                                            int W, int H, int F, const int *sid, TauRec *srec, uint32_t *sbox)
{
    for (int j = threadIdx.x; j < nb; j += NT) {
        const int f = bc.fb ? sid[j] : __ldg(bc.ent + base + j);
        if ((unsigned)f >= (unsigned)F) {     // never expected: bins hold valid face ids
#ifdef BR_DEBUG
            printf("bad face id %d (F=%d) fb=%d n=%d base=%d j=%d nb=%d tile=%d img=%d\n", f, F, (int)bc.fb, bc.n,
                   base, j, nb, blockIdx.x, blockIdx.y);
#endif
            srec[j].fid = -1;
            sbox[j] = EMPTY_BOX;
            atomicOr(bc.status, BLUR_ST_EINTERNAL);
            continue;
        }
        stage_one(bc.rseg + (size_t)f * REC_F4, tau, tc, W, H, srec[j], sbox[j]);
    }
}

template <bool CENSUS>
__device__ __forceinline__ void vis_batch(const TauRec *srec, const uint32_t *sbox, int nb, int base, int wx0,
                                          int wy0, float ul, float vl, float &zbest, int &ebest,
                                          unsigned long long &ncov, unsigned long long &ntest, bool count)
{
    const int lane = threadIdx.x & 31;
    for (int j0 = 0; j0 < nb; j0 += 32) {
        const int j = j0 + lane;
        bool hit = false;
        if (j < nb) {
            const uint32_t bx = sbox[j];
            const int x0 = bx & 0xff, x1 = (bx >> 8) & 0xff, y0 = (bx >> 16) & 0xff, y1 = bx >> 24;
            hit = x0 <= wx0 + 7 && x1 >= wx0 && y0 <= wy0 + 3 && y1 >= wy0;
        }
        unsigned m = __ballot_sync(0xffffffffu, hit);
        while (m) {
            const int k = __ffs(m) - 1;
            m &= m - 1;
            const float4 *rp = reinterpret_cast<const float4 *>(srec + j0 + k);
            const float4 q0 = rp[0], q1 = rp[1], q2 = rp[2];
            const float e0 = edge_eval(q0.x, q0.w, q1.z, ul, vl);
            const float e1 = edge_eval(q0.y, q1.x, q1.w, ul, vl);
            const float e2 = edge_eval(q0.z, q1.y, q2.x, ul, vl);
            const float z = __fmaf_rn(q2.y, ul, __fmaf_rn(q2.z, vl, q2.w));
            const bool cov = fminf(fminf(e0, e1), e2) >= 0.f;
            if (CENSUS && count) { ncov += cov; ntest += 1; }
            if (cov && z < zbest) { zbest = z; ebest = base + j0 + k; }
        }
    }
}

__device__ __forceinline__ void weights(const TauRec &r, float ul, float vl, float w[3])
{
    w[0] = edge_eval(r.a[0], r.b[0], r.g[0], ul, vl) * r.invD;
    w[1] = edge_eval(r.a[1], r.b[1], r.g[1], ul, vl) * r.invD;
    w[2] = edge_eval(r.a[2], r.b[2], r.g[2], ul, vl) * r.invD;
}

__device__ __forceinline__ void tile_ctx(const Tables &t, int tile, TileCtx &tc, int &tx, int &ty)
{
    tx = tile % t.TX;
    ty = tile / t.TX;
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

template <bool CENSUS>
__global__ void __launch_bounds__(NT, 4) k4_raster_fwd(Tables t, float *__restrict__ out, int *__restrict__ ids,
                                                    int ids_k, unsigned long long *census)
{
    __shared__ TauRec srec[CAP];
    __shared__ uint32_t sbox[CAP];
    __shared__ int sid[CAP];
    __shared__ int swsum[NT / 32];
    const int b = blockIdx.y, tile = blockIdx.x;
    const ImgInfo &im = t.imgs[b];
    const int N = im.N, c_begin = im.chunk_begin, c_end = im.chunk_end, sched_off = im.sched_off;
    const long long rec_off = im.rec_off;
    TileCtx tc;
    int tx, ty;
    tile_ctx(t, tile, tc, tx, ty);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wx0 = (warp & 1) * 8, wy0 = (warp >> 1) * 4;
    const int lx = wx0 + (lane & 7), ly = wy0 + (lane >> 3);
    const int px = tc.px0 + lx, py = tc.py0 + ly;
    const bool inimg = px < t.W && py < t.H;
    const float ul = (float)(lx - TW / 2) * tc.sx;
    const float vl = (float)(TH / 2 - ly) * tc.sy;
    const size_t pix = ((size_t)b * t.H + py) * t.W + px;
    float ar = 0.f, ag = 0.f, ab = 0.f, aa = 0.f;
    unsigned long long ncov = 0, ntest = 0, nshade = 0, nstage = 0;

    for (int c = c_begin; c < c_end; ++c) {
        const Chunk ch = t.chunks[c];
        const size_t bi = (size_t)c * t.T + tile;
        const int o = t.off[bi];
        const int n = t.off[bi + 1] - o;
        if (n == 0) {
            if (ids && inimg && ids_k >= ch.k0 && ids_k < ch.k1) ids[pix] = -1;
            continue;
        }
        BinCtx bc;
        bc.status = t.status;
        bc.rseg = t.rec + (size_t)(rec_off + (long long)ch.s * t.F) * REC_F4;
        bc.ent = t.entries + o;
        bc.n = n;
        bc.fb = n > SORTCAP || (long long)o + n > t.cap;
        for (int k = ch.k0; k < ch.k1; ++k) {
            const float tau = t.sched_tau[sched_off + k];
            float zbest = __int_as_float(0x7f800000);
            int ebest = -1;
            bool has = false;
            int bfid = -1;
            float pr = 0.f, pg = 0.f, pb = 0.f;
            int base = 0, fpos = 0;
            while (true) {
                const int nb = next_batch(bc, t.F, tau, tc, t.W, t.H, base, fpos, sid, swsum);
                if (nb == 0) break;
                stage_batch(bc, nb, base, tau, tc, t.W, t.H, t.F, sid, srec, sbox);
                if (CENSUS) nstage += (threadIdx.x < nb) ? (nb - threadIdx.x + NT - 1) / NT : 0;
                __syncthreads();
                vis_batch<CENSUS>(srec, sbox, nb, base, wx0, wy0, ul, vl, zbest, ebest, ncov, ntest, inimg);
                if (ebest >= base) {   // winner changed in this batch: shade now (Eq.9)
                    const TauRec &r = srec[ebest - base];
                    float w[3];
                    weights(r, ul, vl, w);
                    const float4 *fc = t.fcol + 3 * (size_t)r.fid;
                    const float4 c0 = __ldg(fc), c1 = __ldg(fc + 1), c2 = __ldg(fc + 2);
                    pr = __fmaf_rn(w[0], c0.x, __fmaf_rn(w[1], c0.w, w[2] * c1.z));
                    pg = __fmaf_rn(w[0], c0.y, __fmaf_rn(w[1], c1.x, w[2] * c1.w));
                    pb = __fmaf_rn(w[0], c0.z, __fmaf_rn(w[1], c1.y, w[2] * c2.x));
                    has = true;
                    bfid = r.fid;
                }
                base += nb;
                __syncthreads();
            }
            if (has) { ar += pr; ag += pg; ab += pb; aa += 1.f; if (CENSUS) nshade++; }
            if (ids && inimg && k == ids_k) ids[pix] = has ? bfid : -1;
        }
    }
    if (inimg) {
        const float inv = 1.0f / (float)N;
        reinterpret_cast<float4 *>(out)[pix] = make_float4(ar * inv, ag * inv, ab * inv, aa * inv);
    }
    if (CENSUS) {
        atomicAdd(census + 0, ncov);
        atomicAdd(census + 1, inimg ? nshade : 0ull);
        atomicAdd(census + 2, ntest);
        atomicAdd(census + 3, nstage);
    }
}

// ------------------------------------------------------------------ backward
//
// Per (tile, sub-frame): the face's gradient is linear in g = dL/dI_k and w_i(p) is affine in the
// tile-local pixel position, so each face only needs nine moments of g over the pixels it won:
// m0 = sum g, mu = sum u g, mv = sum v g (u, v tile-local).  Then (Eq.9, dw/dv_i = -w_i dw/dp)
//   dL/dc_i = (A_i mu + B_i mv + G_i m0) / |D|
//   dL/dv_i = -( A_i (PA.mu) + B_i (PA.mv) + G_i (PA.m0),  same with PB ) / D^2,
//   PA = sum_j A_j c_j, PB = sum_j B_j c_j  (A, B, G the sign-normalised numerator coefficients).
// The moments are reduced pixel-parallel: the won pixels are counting-sorted by winning slot
// (integer shared-memory atomics), every thread forms the 9 moment terms of one won pixel, a warp
// segmented scan sums runs of equal slots, and each face thread combines its (<= 1 + crossings)
// partial sums and evaluates the closed form.  Every phase is balanced over the CTA.

struct BwdSmem {
    TauRec rec[CAP];
    uint32_t box[CAP];
    int sid[CAP];
    int cnt[CAP];          // won-pixel count per staged slot
    int off[CAP];          // exclusive prefix of cnt
    int key[TW * TH];      // sorted won pixels: slot
    int pix[TW * TH];      //                    pixel
    float mom[9][TW * TH]; // segment partial moments at the run's last position (per warp)
    float4 g[TW * TH];     // dL/dI / N of the tile
    int wsum[NT / 32];
    int total;
};

// block-wide exclusive scan of cnt[0..nb) (nb <= CAP = 2 NT) into off[]; returns the total
__device__ __forceinline__ int scan_counts(BwdSmem &S, int nb)
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
    for (int w = 0; w < NT / 32; ++w) {
        const int v = S.wsum[w];
        pre += w < warp ? v : 0;
        tot += v;
    }
    const int ex = pre + x - (c0 + c1);
    if (j0 < nb) S.off[j0] = ex;
    if (j0 + 1 < nb) S.off[j0 + 1] = ex + c0;
    return tot;
}

struct FaceAcc {
    float k0[6];   // d/d keyframe s position of corners 0..2 (x, y)
    float k1[6];   // d/d keyframe s+1
    float c[9];    // d/d colour of corners 0..2
};

__device__ __forceinline__ void acc_zero(FaceAcc &a)
{
#pragma unroll
    for (int i = 0; i < 6; ++i) { a.k0[i] = 0.f; a.k1[i] = 0.f; }
#pragma unroll
    for (int i = 0; i < 9; ++i) a.c[i] = 0.f;
}

// closed-form face gradient at tau from its moments (see the comment above)
__device__ __forceinline__ void face_grad(const TauRec &r, const float m[9], const float4 *__restrict__ fcol,
                                          float dv[6], float dc[9])
{
    const float m0x = m[0], m0y = m[1], m0z = m[2], mux = m[3], muy = m[4], muz = m[5], mvx = m[6], mvy = m[7],
                mvz = m[8];
    const float4 *fc = fcol + 3 * (size_t)r.fid;
    const float4 c0 = __ldg(fc), c1 = __ldg(fc + 1), c2 = __ldg(fc + 2);
    const float iD = r.invD;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const float A = r.a[i], B = r.b[i], G = r.g[i];
        dc[3 * i + 0] = (A * mux + B * mvx + G * m0x) * iD;
        dc[3 * i + 1] = (A * muy + B * mvy + G * m0y) * iD;
        dc[3 * i + 2] = (A * muz + B * mvz + G * m0z) * iD;
    }
    const float pax = r.a[0] * c0.x + r.a[1] * c0.w + r.a[2] * c1.z;
    const float pay = r.a[0] * c0.y + r.a[1] * c1.x + r.a[2] * c1.w;
    const float paz = r.a[0] * c0.z + r.a[1] * c1.y + r.a[2] * c2.x;
    const float pbx = r.b[0] * c0.x + r.b[1] * c0.w + r.b[2] * c1.z;
    const float pby = r.b[0] * c0.y + r.b[1] * c1.x + r.b[2] * c1.w;
    const float pbz = r.b[0] * c0.z + r.b[1] * c1.y + r.b[2] * c2.x;
    const float qa0 = pax * m0x + pay * m0y + paz * m0z, qau = pax * mux + pay * muy + paz * muz;
    const float qav = pax * mvx + pay * mvy + paz * mvz;
    const float qb0 = pbx * m0x + pby * m0y + pbz * m0z, qbu = pbx * mux + pby * muy + pbz * muz;
    const float qbv = pbx * mvx + pby * mvy + pbz * mvz;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const float A = r.a[i], B = r.b[i], G = r.g[i];
        dv[2 * i + 0] = -((A * qau + B * qav + G * qa0) * iD) * iD;
        dv[2 * i + 1] = -((A * qbu + B * qbv + G * qb0) * iD) * iD;
    }
}

__device__ __forceinline__ void flush(const Tables &t, const ImgInfo &im, int s, int fid, const float k0[6],
                                      const float k1[6], const float c[9], float *dC)
{
    const float4 q = __ldg(t.fcol + 3 * (size_t)fid + 2);
    const int vid[3] = {__float_as_int(q.y), __float_as_int(q.z), __float_as_int(q.w)};
    float2 *d0 = t.dkey + im.key_off + (size_t)s * t.V;
    float2 *d1 = d0 + t.V;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        if (k0[2 * i] != 0.f || k0[2 * i + 1] != 0.f) atomicAdd(d0 + vid[i], make_float2(k0[2 * i], k0[2 * i + 1]));
        if (k1[2 * i] != 0.f || k1[2 * i + 1] != 0.f) atomicAdd(d1 + vid[i], make_float2(k1[2 * i], k1[2 * i + 1]));
        atomicAdd(dC + 3 * vid[i] + 0, c[3 * i + 0]);
        atomicAdd(dC + 3 * vid[i] + 1, c[3 * i + 1]);
        atomicAdd(dC + 3 * vid[i] + 2, c[3 * i + 2]);
    }
}

// Reduce the moments of the won pixels whose winner lies in the staged batch [base, base+nb) and
// hand each face with winners its closed-form gradient: persistent slots (single batch, slot ==
// thread) accumulate in registers across the chunk, the others flush immediately.
__device__ __forceinline__ void bwd_batch(BwdSmem &S, const Tables &t, const ImgInfo &im, int s, float tau, int base,
                                          int nb, bool persist_ok, int ebest, int myp, const TileCtx &tc,
                                          FaceAcc &acc, float *dC)
{
    const int tid = threadIdx.x, lane = tid & 31;
    for (int j = tid; j < nb; j += NT) S.cnt[j] = 0;
    __syncthreads();
    const int e = ebest - base;
    const bool mine = ebest >= 0 && e >= 0 && e < nb;
    int rank = 0;
    if (mine) rank = atomicAdd(&S.cnt[e], 1);
    __syncthreads();
    const int total = scan_counts(S, nb);
    __syncthreads();
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
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int ku = __shfl_up_sync(0xffffffffu, key, d);
            const bool take = lane >= d && ku == key;
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
        const int st = S.off[j], en = st + c - 1;
        float m[9];
#pragma unroll
        for (int q = 0; q < 9; ++q) m[q] = S.mom[q][en];
        for (int i = st | 31; i < en; i += 32)        // partial sums ending at warp boundaries
#pragma unroll
            for (int q = 0; q < 9; ++q) m[q] += S.mom[q][i];
        float dv[6], dc[9];
        face_grad(S.rec[j], m, t.fcol, dv, dc);
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
            flush(t, im, s, S.rec[j].fid, a0, a1, dc, dC);
        }
    }
}

__global__ void __launch_bounds__(NT, 3) k6_raster_bwd(Tables t, const float *__restrict__ grad, float *__restrict__ dC)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    BwdSmem &S = *reinterpret_cast<BwdSmem *>(smem_raw);
    const int b = blockIdx.y, tile = blockIdx.x;
    const ImgInfo &im = t.imgs[b];
    const int N = im.N, c_begin = im.chunk_begin, c_end = im.chunk_end, sched_off = im.sched_off;
    const long long rec_off = im.rec_off;
    TileCtx tc;
    int tx, ty;
    tile_ctx(t, tile, tc, tx, ty);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wx0 = (warp & 1) * 8, wy0 = (warp >> 1) * 4;
    const int lx = wx0 + (lane & 7), ly = wy0 + (lane >> 3);
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
    __syncthreads();
    unsigned long long dummy0 = 0, dummy1 = 0;

    for (int c = c_begin; c < c_end; ++c) {
        const Chunk ch = t.chunks[c];
        const size_t bi = (size_t)c * t.T + tile;
        const int o = t.off[bi];
        const int n = t.off[bi + 1] - o;
        if (n == 0) continue;
        BinCtx bc;
        bc.status = t.status;
        bc.rseg = t.rec + (size_t)(rec_off + (long long)ch.s * t.F) * REC_F4;
        bc.ent = t.entries + o;
        bc.n = n;
        bc.fb = n > SORTCAP || (long long)o + n > t.cap;
        const bool single = !bc.fb && n <= CAP;
        const bool persist = single && (int)threadIdx.x < n;
        FaceAcc acc;
        acc_zero(acc);
        for (int k = ch.k0; k < ch.k1; ++k) {
            const float tau = t.sched_tau[sched_off + k];
            float zbest = __int_as_float(0x7f800000);
            int ebest = -1;
            int base = 0, fpos = 0;
            // visibility (identical to the forward pass)
            while (true) {
                const int nb = next_batch(bc, t.F, tau, tc, t.W, t.H, base, fpos, S.sid, S.wsum);
                if (nb == 0) break;
                stage_batch(bc, nb, base, tau, tc, t.W, t.H, t.F, S.sid, S.rec, S.box);
                __syncthreads();
                vis_batch<false>(S.rec, S.box, nb, base, wx0, wy0, ul, vl, zbest, ebest, dummy0, dummy1, false);
                base += nb;
                __syncthreads();
            }
            if (!inimg) ebest = -1;
            if (single) {
                bwd_batch(S, t, im, ch.s, tau, 0, n, true, ebest, myp, tc, acc, dC);
            } else {
                // several batches: re-stage each batch and flush per sub-frame
                base = 0;
                fpos = 0;
                while (true) {
                    const int nb = next_batch(bc, t.F, tau, tc, t.W, t.H, base, fpos, S.sid, S.wsum);
                    if (nb == 0) break;
                    stage_batch(bc, nb, base, tau, tc, t.W, t.H, t.F, S.sid, S.rec, S.box);
                    __syncthreads();
                    bwd_batch(S, t, im, ch.s, tau, base, nb, false, ebest, myp, tc, acc, dC);
                    base += nb;
                    __syncthreads();
                }
            }
            __syncthreads();
        }
        if (persist) {
            bool nz = false;
#pragma unroll
            for (int i = 0; i < 9; ++i) nz |= acc.c[i] != 0.f;
#pragma unroll
            for (int i = 0; i < 6; ++i) nz |= (acc.k0[i] != 0.f) | (acc.k1[i] != 0.f);
            if (nz) flush(t, im, ch.s, __ldg(bc.ent + threadIdx.x), acc.k0, acc.k1, acc.c, dC);
        }
    }
}

cudaError_t launch_raster_fwd(const Tables &t, float *out, int *ids, int ids_k, unsigned long long *census,
                              cudaStream_t st)
{
    if (t.B == 0 || t.T == 0) return cudaSuccess;
    dim3 grid(t.T, t.B);
    if (census) k4_raster_fwd<true><<<grid, NT, 0, st>>>(t, out, ids, ids_k, census);
    else k4_raster_fwd<false><<<grid, NT, 0, st>>>(t, out, ids, ids_k, nullptr);
    return cudaGetLastError();
}

cudaError_t launch_raster_bwd(const Tables &t, const float *grad, float *dC, cudaStream_t st)
{
    if (t.B == 0 || t.T == 0 || t.F == 0) return cudaSuccess;
    dim3 grid(t.T, t.B);
    const int smem = (int)sizeof(BwdSmem);
    cudaError_t e = cudaFuncSetAttribute(k6_raster_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    k6_raster_bwd<<<grid, NT, smem, st>>>(t, grad, dC);
    return cudaGetLastError();
}

}  // namespace br
