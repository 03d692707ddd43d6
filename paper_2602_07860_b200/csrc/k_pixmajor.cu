// k_pixmajor.cu -- K4 in the pixel-major evaluation order: SURVEY §8(a) a4 order (i), the paper's "the
// coefficients are computed only once and evaluated for K frames" (Eq.7-8) taken literally at the
// pixel.  A measured A/B variant of the forward (BLURRAST_FWD=pixmajor); the timed path is k4l_raster_fwd's
// tau-hoisted order (ii) (k_raster.cu), and DESIGN.md §4 gives the measurements that decided between them.
//
// Order (ii) (k4l): per (face, sub-frame, tile) the Eq.8 numerators are Horner-evaluated in tau into an
// affine edge function of the pixel, and every pixel test is 2 FMA per numerator.  Order (i) (here): per
// (face, chunk, tile) the record is staged once, tile-local, as
//     N_i(tau; p) = A3_i(p) + tau A2_i(p) + tau^2 A1_i          (Eq.8: A1 constant, A2 and A3 affine in p)
// with A3_i(p) = a0 ul + b0 vl + P_i and A2_i(p) = a1 ul + b1 vl + Q_i; per (pixel, face) a lane forms A3_i(p),
// A2_i(p) once (12 FMA), then per sub-frame tau of the chunk evaluates N_i by Horner (2 FMA each) and
// D(tau) = a1 tau^2 + a2 tau + a3 (Eq.8's denominator), tests coverage by sign (all N_i sgn D >= 0)
// and keeps the nearest face per sub-frame in a register z-buffer of KP slots.  Culling: a face enters the
// list of every warp footprint its box swept over the chunk reaches; per (face, tau) a warp-uniform test of
// the face's box at tau against the footprint and of |D(tau)| > EPS_D (Q8) skips the sub-frames it cannot
// cover.  Depth (Q6): z = z_a(tau) + (N_1 (z_b - z_a)(tau) + N_2 (z_c - z_a)(tau)) / D(tau), ties by face
// index (Q7).  Shading (Eq.9) of each sub-frame's winner from its K2 record, accumulated per pixel; the
// blurred image (1/N) sum is written once.  Coverage is watertight for the same reason as in k4l: both faces
// of an edge derive (a0, b0, P, a1, b1, Q, R) from the same canonical K2 edge data with explicit-rounding
// arithmetic, so their numerators are exact negations.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "internal.cuh"
#include "raster_common.cuh"
#include "../../include/blurrast.h"

namespace br {

#ifndef BR_PM_NB
#define BR_PM_NB 256   // faces staged per batch (bins up to VIS_MAXN take one batch)
#endif
#ifndef BR_PM_KP
#define BR_PM_KP 8     // sub-frames per register pass (z-buffer slots per thread)
#endif
#ifndef BR_PM_MINB
#define BR_PM_MINB 4
#endif
constexpr int PM_NB = BR_PM_NB;
constexpr int PM_KP = BR_PM_KP;
constexpr int PM_NW = NT / 32;                 // warps = 8x4 footprints per 16x16 tile
static_assert(PM_NB <= 256 && VIS_MAXN <= PM_NB, "list entries are bytes; cached bins take one batch");

struct __align__(16) PMRec {   // one (face, chunk) record, tile-local: 11 x float4 = 176 B
    float4 e0[3];   // per edge i: (a0, b0, P, a1)
    float4 e1[3];   // per edge i: (b1, Q, R, -)
    float4 d;       // (d1, d2, d3, face id bits): D(tau) = d3 + tau (d2 + tau d1)
    float4 z0, dz;  // view depth of the corners at keyframe s, and keyframe s+1 minus s
    float4 bx0, bx1;   // keyframe boxes (xmin, xmax, ymin, ymax) minus the tile reference centre
};

struct __align__(16) PMSmem {
    PMRec rec[PM_NB];
    uint8_t list[PM_NW][PM_NB];   // per footprint: batch-local indices of the faces whose swept box reaches it
    int cnt[PM_NW];
    float taus[PM_KP];
    float4 acc[TW * TH];          // per-pixel (r, g, b, a) sums over the sub-frames
};

// the tile-local order-(i) coefficients of edge i of a K2 record (identical arithmetic wherever evaluated)
__device__ __forceinline__ void pm_edge(const float *ef, int i, const TileCtx &tc, float &a0, float &b0, float &P,
                                        float &a1, float &b1, float &Q, float &R)
{
    const float ox = ef[8 * i], oy = ef[8 * i + 1];
    a0 = ef[8 * i + 2]; a1 = ef[8 * i + 3];
    b0 = ef[8 * i + 4]; b1 = ef[8 * i + 5];
    const float dax = ef[8 * i + 6], day = ef[8 * i + 7];
    const float dx = __fsub_rn(tc.uc, ox), dy = __fsub_rn(tc.vc, oy);
    // N_i = (a0 + a1 tau)(ul + dx - tau dax) + (b0 + b1 tau)(vl + dy - tau day), expanded in tau (order (i))
    P = __fmaf_rn(a0, dx, __fmul_rn(b0, dy));
    const float g1 = -__fmaf_rn(a0, dax, __fmul_rn(b0, day));
    R = -__fmaf_rn(a1, dax, __fmul_rn(b1, day));
    Q = __fmaf_rn(a1, dx, __fmaf_rn(b1, dy, g1));
}

// N_i at the pixel: A3 + tau (A2 + tau A1)
__device__ __forceinline__ float pm_num(float c0, float c1, float R, float tau)
{
    return __fmaf_rn(tau, __fmaf_rn(tau, R, c1), c0);
}

template <bool COV>
__global__ void __launch_bounds__(NT, BR_PM_MINB) k4i_raster_fwd(Tables t, float *__restrict__ out,
                                                                 int *__restrict__ ids, int ids_k)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    PMSmem &S = *reinterpret_cast<PMSmem *>(smem_raw);
    const int b = blockIdx.y, tile = blockIdx.x;
    const ImgInfo &im = t.imgs[b];
    const int N = im.N, sched_off = im.sched_off;
    TileCtx tc;
    tile_ctx(t, tile, tc);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int fx0 = (warp & 1) * 8, fy0 = (warp >> 1) * 4;
    const int lx = fx0 + (lane & 7), ly = fy0 + (lane >> 3);
    const int px = tc.px0 + lx, py = tc.py0 + ly;
    const bool inimg = px < t.W && py < t.H;
    const float ul = (float)(lx - TW / 2) * tc.sx;
    const float vl = (float)(TH / 2 - ly) * tc.sy;
    const int myp = ly * TW + lx;
    const size_t pix = ((size_t)b * t.H + py) * t.W + px;
    // the warp footprint's pixel-centre extent, tile-local NDC (the boxes carry 1e-5 of padding, far more than
    // the rounding of these bounds: a face culled by them covers no pixel centre of the footprint)
    const float fu0 = (float)(fx0 - TW / 2) * tc.sx, fu1 = (float)(fx0 + 7 - TW / 2) * tc.sx;
    const float fv1 = (float)(TH / 2 - fy0) * tc.sy, fv0 = (float)(TH / 2 - fy0 - 3) * tc.sy;
    S.acc[myp] = make_float4(0.f, 0.f, 0.f, 0.f);

    for (int c = im.chunk_begin + (int)blockIdx.z; c < im.chunk_end; c += t.splits) {
        const Chunk ch = t.chunks[c];
        const size_t bi = (size_t)c * t.T + tile;
        const long long o = t.off[bi];
        int n = (int)(t.off[bi + 1] - o);
        const bool fb = o + n > t.cap;             // overflowed bin: every face of the segment, in index order
        const int *ent = fb ? nullptr : t.entries + o;
        if (fb) n = t.F;
        const float4 *rseg = t.rec + (size_t)(im.rec_off + (long long)ch.s * t.F) * REC_F4;
        uint16_t *vis_out = (!fb && n <= VIS_MAXN) ? t.vis : nullptr;
        const int nbatch = (n + PM_NB - 1) / PM_NB;
        for (int k0 = ch.k0; k0 < ch.k1; k0 += PM_KP) {
            const int kp = min(PM_KP, ch.k1 - k0);
            float zb[PM_KP];
            int jb[PM_KP];
#pragma unroll
            for (int l = 0; l < PM_KP; ++l) { zb[l] = __int_as_float(0x7f800000); jb[l] = -1; }
            for (int bt = 0; bt < nbatch; ++bt) {
                const int base = bt * PM_NB, nb = min(PM_NB, n - base);
                __syncthreads();   // previous batch / pass consumed
                if (threadIdx.x < kp) S.taus[threadIdx.x] = t.sched_tau[sched_off + k0 + threadIdx.x];
                if (threadIdx.x < PM_NW) S.cnt[threadIdx.x] = 0;
                __syncthreads();
                // stage: thread per face of the batch
                const float ta = S.taus[0], tb = S.taus[kp - 1];
                for (int j = threadIdx.x; j < nb; j += NT) {
                    const int f = ent ? __ldg(ent + base + j) : base + j;
                    if ((unsigned)f >= (unsigned)t.F) { atomicOr(t.status, BLUR_ST_EINTERNAL); continue; }
                    FaceRec fr;
                    load_rec(rseg + (size_t)f * REC_F4, fr);
                    if (__float_as_int(fr.q[6].w) < 0) continue;          // skipped face (Q8, behind, bad index)
                    // swept box of the pass (the lerped keyframe boxes are monotone in tau, as in K3)
                    const float4 b0 = fr.q[7], b1 = fr.q[8];
                    int x0, x1, y0, y1;
                    if (!tile_pixels(fminf(box_lerp(ta, b0.x, b1.x), box_lerp(tb, b0.x, b1.x)),
                                     fmaxf(box_lerp(ta, b0.y, b1.y), box_lerp(tb, b0.y, b1.y)),
                                     fminf(box_lerp(ta, b0.z, b1.z), box_lerp(tb, b0.z, b1.z)),
                                     fmaxf(box_lerp(ta, b0.w, b1.w), box_lerp(tb, b0.w, b1.w)), t.W, t.H, tc, x0, x1,
                                     y0, y1))
                        continue;
                    PMRec &R = S.rec[j];
                    const float *ef = reinterpret_cast<const float *>(fr.q);
#pragma unroll
                    for (int i = 0; i < 3; ++i) {
                        float a0, bb0, P, a1, bb1, Q, Rr;
                        pm_edge(ef, i, tc, a0, bb0, P, a1, bb1, Q, Rr);
                        R.e0[i] = make_float4(a0, bb0, P, a1);
                        R.e1[i] = make_float4(bb1, Q, Rr, 0.f);
                    }
                    R.d = fr.q[6];
                    const float4 z0 = fr.q[9], z1 = fr.q[10];
                    R.z0 = z0;
                    R.dz = make_float4(z1.x - z0.x, z1.y - z0.y, z1.z - z0.z, 0.f);
                    R.bx0 = make_float4(b0.x - tc.uc, b0.y - tc.uc, b0.z - tc.vc, b0.w - tc.vc);
                    R.bx1 = make_float4(b1.x - tc.uc, b1.y - tc.uc, b1.z - tc.vc, b1.w - tc.vc);
                    for (int wy = y0 >> 2; wy <= (y1 >> 2); ++wy)
                        for (int wx = x0 >> 3; wx <= (x1 >> 3); ++wx) {
                            const int w = wy * 2 + wx;
                            S.list[w][atomicAdd(&S.cnt[w], 1)] = (uint8_t)j;
                        }
                }
                __syncthreads();
                // vis: the warp's footprint list, every face at each sub-frame of the pass
                const int cn = S.cnt[warp];
                for (int e = 0; e < cn; ++e) {
                    const int j = S.list[warp][e];
                    const PMRec &R = S.rec[j];
                    const float4 d = R.d, bx0 = R.bx0, bx1 = R.bx1;
                    unsigned tm = 0u;   // warp-uniform: sub-frames whose box reaches the footprint, |D| > EPS_D
#pragma unroll
                    for (int l = 0; l < PM_KP; ++l) {
                        if (l < kp) {
                            const float tau = S.taus[l];
                            // box at tau, relative to the tile centre (box_lerp of the shifted keyframe boxes;
                            // the shift is far below the 1e-5 box padding)
                            const bool hit = box_lerp(tau, bx0.x, bx1.x) <= fu1 && box_lerp(tau, bx0.y, bx1.y) >= fu0 &&
                                             box_lerp(tau, bx0.z, bx1.z) <= fv1 && box_lerp(tau, bx0.w, bx1.w) >= fv0;
                            const float D = __fmaf_rn(tau, __fmaf_rn(tau, d.x, d.y), d.z);
                            if (hit && fabsf(D) > EPS_D) tm |= 1u << l;
                        }
                    }
                    if (!tm) continue;
                    float c0[3], c1[3], Rr[3];
#pragma unroll
                    for (int i = 0; i < 3; ++i) {
                        const float4 p = R.e0[i], q = R.e1[i];
                        c0[i] = __fmaf_rn(p.x, ul, __fmaf_rn(p.y, vl, p.z));   // A3_i(p)
                        c1[i] = __fmaf_rn(p.w, ul, __fmaf_rn(q.x, vl, q.y));   // A2_i(p)
                        Rr[i] = q.z;                                           // A1_i
                    }
#pragma unroll
                    for (int l = 0; l < PM_KP; ++l) {
                        if (!((tm >> l) & 1u)) continue;
                        const float tau = S.taus[l];
                        const float D = __fmaf_rn(tau, __fmaf_rn(tau, d.x, d.y), d.z);
                        const float n0 = pm_num(c0[0], c1[0], Rr[0], tau);
                        const float n1 = pm_num(c0[1], c1[1], Rr[1], tau);
                        const float n2 = pm_num(c0[2], c1[2], Rr[2], tau);
                        const bool cov = D > 0.f ? fminf(fminf(n0, n1), n2) >= 0.f : fmaxf(fmaxf(n0, n1), n2) <= 0.f;
                        if (cov) {
                            const float4 z0 = R.z0, dz = R.dz;
                            const float za = __fmaf_rn(tau, dz.x, z0.x);
                            const float zbv = __fmaf_rn(tau, dz.y, z0.y) - za;
                            const float zcv = __fmaf_rn(tau, dz.z, z0.z) - za;
                            const float z = __fmaf_rn(__fmaf_rn(n1, zbv, __fmul_rn(n2, zcv)), __frcp_rn(D), za);
                            const int jg = base + j;
                            bool take = z < zb[l];
                            if (z == zb[l] && jb[l] >= 0) {   // exact depth tie: the lower face index wins (Q7)
                                const int fw = ent ? __ldg(ent + jb[l]) : jb[l];
                                const int fc = __float_as_int(d.w);
                                take = fc < fw;
                            }
                            if (take) { zb[l] = z; jb[l] = jg; }
                        }
                    }
                }
            }
            // shade the pass's sub-frames from the winners' K2 records (Eq.9) and accumulate
#pragma unroll
            for (int l = 0; l < PM_KP; ++l) {
                if (l >= kp) continue;
                const int k = k0 + l;
                int fid = -1;
                if (jb[l] >= 0) {
                    const float tau = t.sched_tau[sched_off + k];
                    const int f = ent ? __ldg(ent + jb[l]) : jb[l];
                    const float4 *rp = rseg + (size_t)f * REC_F4;
                    float4 q[7];
#pragma unroll
                    for (int i = 0; i < 7; ++i) q[i] = __ldg(rp + i);
                    const float *ef = reinterpret_cast<const float *>(q);
                    float w[3];
                    const float D = __fmaf_rn(tau, __fmaf_rn(tau, q[6].x, q[6].y), q[6].z);
                    const float iD = __frcp_rn(D);
#pragma unroll
                    for (int i = 0; i < 3; ++i) {
                        float a0, bb0, P, a1, bb1, Q, Rr;
                        pm_edge(ef, i, tc, a0, bb0, P, a1, bb1, Q, Rr);
                        const float c0 = __fmaf_rn(a0, ul, __fmaf_rn(bb0, vl, P));
                        const float c1 = __fmaf_rn(a1, ul, __fmaf_rn(bb1, vl, Q));
                        w[i] = pm_num(c0, c1, Rr, tau) * iD;
                    }
                    fid = f;
                    const float4 *fc = t.fcol + 3 * (size_t)f;
                    const float4 q0 = __ldg(fc), q1 = __ldg(fc + 1), q2 = __ldg(fc + 2);
                    float4 a = S.acc[myp];
                    a.x += __fmaf_rn(w[0], q0.x, __fmaf_rn(w[1], q0.w, w[2] * q1.z));
                    a.y += __fmaf_rn(w[0], q0.y, __fmaf_rn(w[1], q1.x, w[2] * q1.w));
                    a.z += __fmaf_rn(w[0], q0.z, __fmaf_rn(w[1], q1.y, w[2] * q2.x));
                    a.w += 1.f;
                    S.acc[myp] = a;
                }
                if (ids && inimg && k == ids_k) ids[pix] = fid;
                if (vis_out)
                    vis_out[((size_t)(im.cov_off + k) * t.T + tile) * (TW * TH) + myp] =
                        jb[l] >= 0 ? (uint16_t)jb[l] : (uint16_t)0xFFFF;
                if (COV) {
                    const unsigned m = __ballot_sync(0xffffffffu, jb[l] >= 0 || !inimg);
                    if (lane == 0) t.covbits[cov_word(t, im, k, tile) + warp] = m;
                }
            }
        }
    }
    if (inimg && out) {
        const float inv = 1.0f / (float)N;
        const float4 a = S.acc[myp];
        const float4 v = make_float4(a.x * inv, a.y * inv, a.z * inv, a.w * inv);
        if (t.splits == 1) reinterpret_cast<float4 *>(out)[pix] = v;
        else t.part[(size_t)blockIdx.z * ((size_t)t.B * t.H * t.W) + pix] = v;
    }
}

template <bool COV>
static cudaError_t launch_pm(const Tables &t, float *out, int *ids, int ids_k, cudaStream_t st)
{
    dim3 grid(t.T, t.B, t.splits);
    const int smem = (int)sizeof(PMSmem);
    cudaError_t e = cudaFuncSetAttribute(k4i_raster_fwd<COV>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    k4i_raster_fwd<COV><<<grid, NT, smem, st>>>(t, out, ids, ids_k);
    return cudaGetLastError();
}

bool pixmajor_fwd_on()
{
    const char *s = std::getenv("BLURRAST_FWD");
    return s && std::strcmp(s, "pixmajor") == 0;
}

cudaError_t launch_raster_fwd_pixmajor(const Tables &t, float *out, int *ids, int ids_k, cudaStream_t st)
{
    if (t.B == 0 || t.T == 0) return cudaSuccess;
    return t.covbits ? launch_pm<true>(t, out, ids, ids_k, st) : launch_pm<false>(t, out, ids, ids_k, st);
}

}  // namespace br
