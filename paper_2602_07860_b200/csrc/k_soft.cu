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
// Which (pixel, sub-frame) are background comes from the hard raster pass (K4), which leaves one
// coverage ballot per (sub-frame, tile, warp) in the workspace (1 bit per pixel and sub-frame).
// The soft kernels use their own bins (K3 on the chunk boxes grown by rcut, faces in index order).
//   K8 (fwd)  CTA = 16x16 tile, 8 warps of 8x4 pixels.  Per group of sub-frames: every
//             (face, tau) pair whose grown box reaches the tile is staged once into a 96 B
//             shared-memory record (w(tau) coefficients, F(X) and F(tau) tile-local vertices,
//             inverse squared F(X) edge lengths) with a per-(tau, warp) bit mask of the warp
//             footprints that need it (uncovered pixels within rcut of the face at tau); every
//             uncovered lane then folds its faces into prod (1 - A) in registers, in face order.
//             The per-split partial alphas are reduced in a fixed order (deterministic).
//   K9 (bwd)  w^* frozen: dalpha/dA_j = prod_{l != j} (1 - A_l), dA/dd = -A/delta,
//             dd/dv_i(tau) = -2 w^*_i (p - F(tau) w^*).  Pass 1 (pixel-parallel) recomputes the
//             product per background pixel; pass 2 (face-parallel: one thread per staged face)
//             walks the needing pixels of the face's warp footprints and accumulates the face's
//             corner gradients in registers over the chunk, split (1 - tau, tau) onto keyframes and
//             flushed with one vector RED per (corner, keyframe).
#include <algorithm>
#include <cstdio>

#include "internal.cuh"
#include "../../include/blurrast.h"

namespace br {

namespace {

constexpr int SNW = NT / 32;     // warps per CTA
constexpr int SREC_S = 512;      // staged soft records per CTA (96 B each)
constexpr int GMAX_S = 8;        // sub-frames staged together
constexpr int NPX = TW * TH;

struct __align__(16) SoftRec {
    // q0: wa0 wa1 wa2 wb0 | q1: wb1 wb2 wg0 wg1 | q2: wg2 xX0 yX0 xX1 | q3: yX1 xX2 yX2 il01
    // q4: il12 il20 xT0 yT0 | q5: xT1 yT1 xT2 yT2       (w_i = wa_i ul + wb_i vl + wg_i)
    float4 q[6];
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
__device__ __forceinline__ bool rect_near(const float A[3], const float B[3], const float G[3], int x0, int x1,
                                          int y0, int y1, float rcut, const STile &tc)
{
    const float ulmin = (float)(x0 - TW / 2) * tc.sx, ulmax = (float)(x1 - TW / 2) * tc.sx;
    const float vlmin = (float)(TH / 2 - y1) * tc.sy, vlmax = (float)(TH / 2 - y0) * tc.sy;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const float m = G[i] + (A[i] > 0.f ? A[i] * ulmax : A[i] * ulmin) + (B[i] > 0.f ? B[i] * vlmax : B[i] * vlmin);
        const float nrm = sqrtf(A[i] * A[i] + B[i] * B[i]);
        const float tol = 1e-5f * (fabsf(A[i]) * fmaxf(-ulmin, ulmax) + fabsf(B[i]) * fmaxf(-vlmin, vlmax) +
                                   fabsf(G[i])) + 1e-30f;
        if (m < -(rcut * nrm) - tol) return false;
    }
    return true;
}

// Stage one (face, tau) soft record for this tile.  need[w] = uncovered-pixel bits of warp w at
// tau.  Returns the mask of warp footprints the record must visit (0 = none).
__device__ __forceinline__ uint32_t soft_stage(const Tables &t, const float4 *__restrict__ r,
                                               const float4 *__restrict__ key0, const float4 *__restrict__ key1,
                                               int f, float tau, const STile &tc, const uint32_t *need,
                                               SoftRec &out)
{
    const float4 q6 = __ldg(r + 6);
    if (__float_as_int(q6.w) < 0) return 0u;                             // skipped face
    const float D = __fmaf_rn(tau, __fmaf_rn(tau, q6.x, q6.y), q6.z);   // det F(tau) (Eq.8 a-coefficients)
    if (!(fabsf(D) > EPS_D)) return 0u;                                 // Q8
    int x0, x1, y0, y1;
    if (!grown_box(r, tau, t.rcut, t.W, t.H, tc, x0, x1, y0, y1)) return 0u;
    const float sg = D < 0.f ? -1.f : 1.f;
    const float invD = 1.0f / fabsf(D);
    float A[3], B[3], G[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {   // Eq.8 numerators at tau, re-centred at the tile centre
        const float4 e0 = __ldg(r + 2 * i), e1 = __ldg(r + 2 * i + 1);   // ox oy a0 a1 | b0 b1 g1 g2
        const float al = __fmaf_rn(tau, e0.w, e0.z);
        const float be = __fmaf_rn(tau, e1.y, e1.x);
        const float ga = __fmul_rn(tau, __fmaf_rn(tau, e1.w, e1.z));
        const float dx = __fsub_rn(tc.uc, e0.x), dy = __fsub_rn(tc.vc, e0.y);
        const float gp = __fmaf_rn(al, dx, __fmaf_rn(be, dy, ga));
        A[i] = al * sg;
        B[i] = be * sg;
        G[i] = gp * sg;
    }
    uint32_t fm = 0u;
    for (int wy = y0 >> 2; wy <= (y1 >> 2); ++wy)
        for (int wx = x0 >> 3; wx <= (x1 >> 3); ++wx) {
            const int w = wy * 2 + wx;
            if (!need[w]) continue;
            const int rx0 = max(x0, wx * 8), rx1 = min(x1, wx * 8 + 7);
            const int ry0 = max(y0, wy * 4), ry1 = min(y1, wy * 4 + 3);
            if (rect_near(A, B, G, rx0, rx1, ry0, ry1, t.rcut, tc)) fm |= 1u << w;
        }
    if (!fm) return 0u;
    const float4 vc = __ldg(t.fcol + 3 * (size_t)f + 2);
    const int vid[3] = {__float_as_int(vc.y), __float_as_int(vc.z), __float_as_int(vc.w)};
    float xT[3], yT[3], xX[3], yX[3];
    const bool useX1 = tau > 0.5f;                                      // Eq.13: X = 1 iff tau > 0.5
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const float4 a = __ldg(key0 + vid[i]), b = __ldg(key1 + vid[i]);
        xT[i] = __fsub_rn(__fmaf_rn(tau, __fsub_rn(b.x, a.x), a.x), tc.uc);   // F(tau), Eq.5-6
        yT[i] = __fsub_rn(__fmaf_rn(tau, __fsub_rn(b.y, a.y), a.y), tc.vc);
        if (t.soft_exact) {                                                // Eq.12: F(X) = F(tau)
            xX[i] = xT[i];
            yX[i] = yT[i];
        } else {
            xX[i] = __fsub_rn(useX1 ? b.x : a.x, tc.uc);
            yX[i] = __fsub_rn(useX1 ? b.y : a.y, tc.vc);
        }
    }
    float il[3];
#pragma unroll
    for (int e = 0; e < 3; ++e) {   // edges v0v1, v1v2, v2v0 of F(X) (A17)
        const int j = (e + 1) % 3;
        const float ex = xX[j] - xX[e], ey = yX[j] - yX[e];
        const float l2 = ex * ex + ey * ey;
        il[e] = l2 > 0.f ? 1.0f / l2 : 0.f;   // zero-length edge: t = 0, its vertex (Q19)
    }
    out.q[0] = make_float4(A[0] * invD, A[1] * invD, A[2] * invD, B[0] * invD);
    out.q[1] = make_float4(B[1] * invD, B[2] * invD, G[0] * invD, G[1] * invD);
    out.q[2] = make_float4(G[2] * invD, xX[0], yX[0], xX[1]);
    out.q[3] = make_float4(yX[1], xX[2], yX[2], il[0]);
    out.q[4] = make_float4(il[1], il[2], xT[0], yT[0]);
    out.q[5] = make_float4(xT[1], yT[1], xT[2], yT[2]);
    return fm;
}

// One (pixel, face, tau) term: d (Eq.14) and the chosen edge (e: corners e, (e+1)%3) / parameter t.
struct SoftHit {
    float d, t, psx, psy;
    int e;
};

__device__ __forceinline__ SoftHit soft_eval(const SoftRec &r, float ul, float vl)
{
    const float4 q0 = r.q[0], q1 = r.q[1], q2 = r.q[2], q3 = r.q[3], q4 = r.q[4], q5 = r.q[5];
    // w(tau) (fast solver, Eq.8) and p' = F(X) w(tau) (Eq.13)
    const float w0 = __fmaf_rn(q0.x, ul, __fmaf_rn(q0.w, vl, q1.z));
    const float w1 = __fmaf_rn(q0.y, ul, __fmaf_rn(q1.x, vl, q1.w));
    const float w2 = __fmaf_rn(q0.z, ul, __fmaf_rn(q1.y, vl, q2.x));
    const float xX[3] = {q2.y, q2.w, q3.y}, yX[3] = {q2.z, q3.x, q3.z}, il[3] = {q3.w, q4.x, q4.y};
    const float px = __fmaf_rn(w0, xX[0], __fmaf_rn(w1, xX[1], w2 * xX[2]));
    const float py = __fmaf_rn(w0, yX[0], __fmaf_rn(w1, yX[1], w2 * yX[2]));
    // closest point on F(X): three edge projections, clamped (A17-A18), smallest distance (first on ties)
    float best = __int_as_float(0x7f800000), bt = 0.f;
    int be = 0;
#pragma unroll
    for (int e = 0; e < 3; ++e) {
        const int j = (e + 1) % 3;
        const float ex = xX[j] - xX[e], ey = yX[j] - yX[e];
        const float dx = px - xX[e], dy = py - yX[e];
        const float tt = __saturatef(__fmaf_rn(dx, ex, dy * ey) * il[e]);
        const float rx = __fmaf_rn(-tt, ex, dx), ry = __fmaf_rn(-tt, ey, dy);
        const float dd = __fmaf_rn(rx, rx, ry * ry);
        if (dd < best) { best = dd; bt = tt; be = e; }
    }
    // F(tau) w^* (Eq.14)
    const float xT[3] = {q4.z, q5.x, q5.z}, yT[3] = {q4.w, q5.y, q5.w};
    float xa = xT[0], ya = yT[0], xb = xT[1], yb = yT[1];
    if (be == 1) { xa = xT[1]; ya = yT[1]; xb = xT[2]; yb = yT[2]; }
    else if (be == 2) { xa = xT[2]; ya = yT[2]; xb = xT[0]; yb = yT[0]; }
    SoftHit h;
    h.psx = __fmaf_rn(bt, xb - xa, xa);
    h.psy = __fmaf_rn(bt, yb - ya, ya);
    const float ddx = ul - h.psx, ddy = vl - h.psy;
    h.d = __fmaf_rn(ddx, ddx, ddy * ddy);
    h.t = bt;
    h.e = be;
    return h;
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

// Stage faces [base, base + nb) of the bin (or sid[] in fallback mode) at the ng sub-frames taus:
// records rec[l * nb + j], masks wm[(l * SNW + w) * nw + j / 32] (cleared by the caller).
__device__ __forceinline__ void soft_stage_group(const Tables &t, const SoftBin &sb, int nb, int base, const float *taus,
                                                 int ng, const STile &tc, const uint32_t (*need)[SNW], const int *sid,
                                                 SoftRec *rec, uint32_t *wm)
{
    const int nw = (nb + 31) >> 5;
    for (int p = threadIdx.x; p < nb * ng; p += NT) {
        const int j = p / ng, l = p - j * ng;
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
                                       rec[l * nb + j]);
        const uint32_t bit = 0x80000000u >> (j & 31);
        for (uint32_t m = fm; m; m &= m - 1) atomicOr(wm + (l * SNW + (__ffs(m) - 1)) * nw + (j >> 5), bit);
    }
}

// prod over the masked faces of (1 - A) for this lane's pixel (face order), with the product of
// the non-zero factors and the count of zero factors (for dalpha/dA in the backward)
__device__ __forceinline__ void soft_product(const SoftRec *rec, const uint32_t *wm, int nw, float ul, float vl,
                                             float kexp, float &P, float &Pnz, int &nz)
{
    for (int wd = 0; wd < nw; ++wd) {
        uint32_t m = wm[wd];
        while (m) {
            const int k = __clz(m);
            m ^= 0x80000000u >> k;
            const SoftHit h = soft_eval(rec[(wd << 5) + k], ul, vl);
            const float A = __expf(-h.d * kexp);                     // Eq.10 with the exp kernel (A20)
            const float fac = 1.0f - A;
            P *= fac;                                                // Eq.15
            if (fac == 0.f) nz++;
            else Pnz *= fac;
        }
    }
}

__device__ __forceinline__ void load_need(const Tables &t, const ImgInfo &im, int k, int tile, int warp, int lane,
                                          bool extra, uint32_t *dst)
{
    const uint32_t cov = t.covbits[cov_word(t, im, k, tile) + warp];
    const unsigned m = __ballot_sync(0xffffffffu, !((cov >> lane) & 1u) && extra);
    if (lane == 0) *dst = m;
}

struct SoftFwdSmem {
    SoftRec rec[SREC_S];
    uint32_t wm[GMAX_S * SNW * (SREC_S / 32 + 1)];
    uint32_t need[GMAX_S][SNW];
    int sid[SREC_S];
    float taus[GMAX_S];
    int wsum[SNW];
};

__global__ void __launch_bounds__(NT, 2) k8_soft_fwd(Tables t)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SoftFwdSmem &S = *reinterpret_cast<SoftFwdSmem *>(smem_raw);
    const int b = blockIdx.y, tile = blockIdx.x;
    const ImgInfo &im = t.imgs[b];
    STile tc;
    stile(t, tile, tc);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int lx = (warp & 1) * 8 + (lane & 7), ly = (warp >> 1) * 4 + (lane >> 3);
    const int px = tc.px0 + lx, py = tc.py0 + ly;
    const bool inimg = px < t.W && py < t.H;
    const float ul = (float)(lx - TW / 2) * tc.sx;
    const float vl = (float)(TH / 2 - ly) * tc.sy;
    const float kexp = 1.0f / t.delta;
    float alpha = 0.f;

    for (int c = im.chunk_begin + (int)blockIdx.z; c < im.chunk_end; c += t.splits) {
        const Chunk ch = t.chunks[c];
        SoftBin sb;
        soft_bin(t, im, ch, c, tile, sb);
        if (sb.n == 0) continue;   // no face within rcut of the tile during the chunk: every P = 1
        if (!sb.fb && sb.n <= SREC_S) {
            const int n = sb.n, Gs = min(GMAX_S, SREC_S / n), nw = (n + 31) >> 5;
            for (int kg = ch.k0; kg < ch.k1; kg += Gs) {
                const int ng = min(Gs, ch.k1 - kg);
                for (int l = 0; l < ng; ++l) load_need(t, im, kg + l, tile, warp, lane, inimg, &S.need[l][warp]);
                for (int i = threadIdx.x; i < ng * SNW * nw; i += NT) S.wm[i] = 0u;
                if (threadIdx.x < ng) S.taus[threadIdx.x] = t.sched_tau[im.sched_off + kg + threadIdx.x];
                __syncthreads();
                soft_stage_group(t, sb, n, 0, S.taus, ng, tc, S.need, S.sid, S.rec, S.wm);
                __syncthreads();
                for (int l = 0; l < ng; ++l) {
                    if (!((S.need[l][warp] >> lane) & 1u)) continue;
                    float P = 1.f, Pnz = 1.f;
                    int nz = 0;
                    soft_product(S.rec + l * n, S.wm + (l * SNW + warp) * nw, nw, ul, vl, kexp, P, Pnz, nz);
                    alpha += 1.f - P;
                }
                __syncthreads();
            }
        } else {
            for (int k = ch.k0; k < ch.k1; ++k) {
                load_need(t, im, k, tile, warp, lane, inimg, &S.need[0][warp]);
                if (threadIdx.x == 0) S.taus[0] = t.sched_tau[im.sched_off + k];
                __syncthreads();
                uint32_t anyn = 0u;
#pragma unroll
                for (int w = 0; w < SNW; ++w) anyn |= S.need[0][w];
                const bool mine = (S.need[0][warp] >> lane) & 1u;
                float P = 1.f, Pnz = 1.f;
                int nz = 0;
                int base = 0, fpos = 0;
                while (anyn) {
                    const int nb = sb.fb ? soft_fallback_fill(t, sb.rseg, S.taus[0], tc, SREC_S, fpos, S.sid, S.wsum)
                                         : (base < sb.n ? min(SREC_S, sb.n - base) : 0);
                    if (nb == 0) break;
                    const int nw = (nb + 31) >> 5;
                    for (int i = threadIdx.x; i < SNW * nw; i += NT) S.wm[i] = 0u;
                    __syncthreads();
                    soft_stage_group(t, sb, nb, base, S.taus, 1, tc, S.need, S.sid, S.rec, S.wm);
                    __syncthreads();
                    if (mine) soft_product(S.rec, S.wm + warp * nw, nw, ul, vl, kexp, P, Pnz, nz);
                    base += nb;
                    __syncthreads();
                }
                if (mine) alpha += 1.f - P;
                __syncthreads();
            }
        }
    }
    if (inimg) t.spart[(size_t)blockIdx.z * ((size_t)t.B * t.H * t.W) + ((size_t)b * t.H + py) * t.W + px] =
        alpha / (float)im.N;
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
    SoftRec rec[SREC_S];
    uint32_t wm[GMAX_S * SNW * (SREC_S / 32 + 1)];
    uint32_t need[GMAX_S][SNW];
    float pnz[GMAX_S][NPX];
    int nz[GMAX_S][NPX];
    float ga[NPX];
    int sid[SREC_S];
    float taus[GMAX_S];
    int wsum[SNW];
};

__device__ __forceinline__ void soft_flush(const Tables &t, const ImgInfo &im, int s, int f, const float k0[6],
                                           const float k1[6])
{
    const float4 q = __ldg(t.fcol + 3 * (size_t)f + 2);
    const int vid[3] = {__float_as_int(q.y), __float_as_int(q.z), __float_as_int(q.w)};
    float2 *d0 = t.dkey + im.key_off + (size_t)s * t.V;
    float2 *d1 = d0 + t.V;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        if (k0[2 * i] != 0.f || k0[2 * i + 1] != 0.f) atomicAdd(d0 + vid[i], make_float2(k0[2 * i], k0[2 * i + 1]));
        if (k1[2 * i] != 0.f || k1[2 * i + 1] != 0.f) atomicAdd(d1 + vid[i], make_float2(k1[2 * i], k1[2 * i + 1]));
    }
}

// Face-parallel gradient of the staged records rec[l * nb + j] (j from this thread) at the ng
// sub-frames: corner gradients accumulated over the needing pixels of the masked footprints.
// Slot j == thread persists in acc (acc0/acc1, keyframes s / s+1); others flush immediately.
__device__ __forceinline__ void soft_grad_group(SoftBwdSmem &S, const Tables &t, const ImgInfo &im, int s, int nb,
                                                int ng, const STile &tc, int slot_base, bool persist_ok,
                                                float acc0[6], float acc1[6], const int *fid_of)
{
    const int nw = (nb + 31) >> 5;
    const float kexp = 1.0f / t.delta, c2 = 2.0f / t.delta;
    for (int j = threadIdx.x; j < nb; j += NT) {
        float a0[6], a1[6];
#pragma unroll
        for (int i = 0; i < 6; ++i) { a0[i] = 0.f; a1[i] = 0.f; }
        bool any = false;
        for (int l = 0; l < ng; ++l) {
            const SoftRec &r = S.rec[l * nb + j];
            float dv[6];
#pragma unroll
            for (int i = 0; i < 6; ++i) dv[i] = 0.f;
            bool hit = false;
            for (int w = 0; w < SNW; ++w) {
                if (!((S.wm[(l * SNW + w) * nw + (j >> 5)] << (j & 31)) & 0x80000000u)) continue;
                uint32_t m = S.need[l][w];
                while (m) {
                    const int ln = __ffs(m) - 1;
                    m &= m - 1;
                    const int lx = (w & 1) * 8 + (ln & 7), ly = (w >> 1) * 4 + (ln >> 3), p = ly * TW + lx;
                    const float ul = (float)(lx - TW / 2) * tc.sx;
                    const float vl = (float)(TH / 2 - ly) * tc.sy;
                    const SoftHit h = soft_eval(r, ul, vl);
                    const float A = __expf(-h.d * kexp);
                    if (A == 0.f) continue;
                    const float fac = 1.0f - A;
                    const int z = S.nz[l][p];
                    const float pz = S.pnz[l][p];
                    const float dadA = z == 0 ? pz / fac : ((z == 1 && fac == 0.f) ? pz : 0.f);
                    // dL/dv_i(tau) = G_a dalpha/dA (A/delta) 2 w^*_i (p - F(tau) w^*)
                    const float cc = S.ga[p] * dadA * A * c2;
                    const float gx = cc * (ul - h.psx), gy = cc * (vl - h.psy);
                    const int ia = h.e, ib = h.e == 2 ? 0 : h.e + 1;
                    const float wa = 1.f - h.t, wb = h.t;
#pragma unroll
                    for (int q = 0; q < 3; ++q) {
                        const float wq = (q == ia ? wa : 0.f) + (q == ib ? wb : 0.f);
                        dv[2 * q] = __fmaf_rn(wq, gx, dv[2 * q]);
                        dv[2 * q + 1] = __fmaf_rn(wq, gy, dv[2 * q + 1]);
                    }
                    hit = true;
                }
            }
            if (!hit) continue;
            any = true;
            const float tau = S.taus[l];
#pragma unroll
            for (int i = 0; i < 6; ++i) {
                a0[i] = __fmaf_rn(1.f - tau, dv[i], a0[i]);
                a1[i] = __fmaf_rn(tau, dv[i], a1[i]);
            }
        }
        if (!any) continue;
        if (persist_ok && j == (int)threadIdx.x) {
#pragma unroll
            for (int i = 0; i < 6; ++i) { acc0[i] += a0[i]; acc1[i] += a1[i]; }
        } else {
            soft_flush(t, im, s, fid_of[j + slot_base], a0, a1);
        }
    }
}

__global__ void __launch_bounds__(NT, 2) k9_soft_bwd(Tables t, const float *__restrict__ grad)
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
    const float ul = (float)(lx - TW / 2) * tc.sx;
    const float vl = (float)(TH / 2 - ly) * tc.sy;
    const float kexp = 1.0f / t.delta;
    const float ga = inimg ? __ldg(grad + 4 * (((size_t)b * t.H + py) * t.W + px) + 3) / (float)im.N : 0.f;
    S.ga[myp] = ga;
    const bool want = inimg && ga != 0.f;
    __syncthreads();

    for (int c = im.chunk_begin + (int)blockIdx.z; c < im.chunk_end; c += t.splits) {
        const Chunk ch = t.chunks[c];
        SoftBin sb;
        soft_bin(t, im, ch, c, tile, sb);
        if (sb.n == 0) continue;
        float acc0[6], acc1[6];
#pragma unroll
        for (int i = 0; i < 6; ++i) { acc0[i] = 0.f; acc1[i] = 0.f; }
        const bool grouped = !sb.fb && sb.n <= SREC_S;
        if (grouped) {
            const int n = sb.n, Gs = min(GMAX_S, SREC_S / n), nw = (n + 31) >> 5;
            for (int kg = ch.k0; kg < ch.k1; kg += Gs) {
                const int ng = min(Gs, ch.k1 - kg);
                for (int l = 0; l < ng; ++l) load_need(t, im, kg + l, tile, warp, lane, want, &S.need[l][warp]);
                for (int i = threadIdx.x; i < ng * SNW * nw; i += NT) S.wm[i] = 0u;
                if (threadIdx.x < ng) S.taus[threadIdx.x] = t.sched_tau[im.sched_off + kg + threadIdx.x];
                __syncthreads();
                uint32_t anyn = 0u;
                for (int l = 0; l < ng; ++l)
#pragma unroll
                    for (int w = 0; w < SNW; ++w) anyn |= S.need[l][w];
                if (anyn) {   // block-uniform
                    soft_stage_group(t, sb, n, 0, S.taus, ng, tc, S.need, S.sid, S.rec, S.wm);
                    __syncthreads();
                    for (int l = 0; l < ng; ++l) {          // pass 1: products per background pixel
                        if (!((S.need[l][warp] >> lane) & 1u)) continue;
                        float P = 1.f, Pnz = 1.f;
                        int nz = 0;
                        soft_product(S.rec + l * n, S.wm + (l * SNW + warp) * nw, nw, ul, vl, kexp, P, Pnz, nz);
                        S.pnz[l][myp] = Pnz;
                        S.nz[l][myp] = nz;
                    }
                    __syncthreads();
                    soft_grad_group(S, t, im, ch.s, n, ng, tc, 0, true, acc0, acc1, sb.ent);   // pass 2
                }
                __syncthreads();
            }
            if ((int)threadIdx.x < sb.n) {
                bool nzf = false;
#pragma unroll
                for (int i = 0; i < 6; ++i) nzf |= (acc0[i] != 0.f) | (acc1[i] != 0.f);
                if (nzf) soft_flush(t, im, ch.s, __ldg(sb.ent + threadIdx.x), acc0, acc1);
            }
        } else {
            for (int k = ch.k0; k < ch.k1; ++k) {
                load_need(t, im, k, tile, warp, lane, want, &S.need[0][warp]);
                if (threadIdx.x == 0) S.taus[0] = t.sched_tau[im.sched_off + k];
                __syncthreads();
                uint32_t anyn = 0u;
#pragma unroll
                for (int w = 0; w < SNW; ++w) anyn |= S.need[0][w];
                __syncthreads();       // every warp has read need[] before the next sub-frame rewrites it
                if (!anyn) continue;   // block-uniform
                const bool mine = (S.need[0][warp] >> lane) & 1u;
                float P = 1.f, Pnz = 1.f;
                int nz = 0;
                int base = 0, fpos = 0;
                while (true) {   // pass 1 over all batches
                    const int nb = sb.fb ? soft_fallback_fill(t, sb.rseg, S.taus[0], tc, SREC_S, fpos, S.sid, S.wsum)
                                         : (base < sb.n ? min(SREC_S, sb.n - base) : 0);
                    if (nb == 0) break;
                    const int nw = (nb + 31) >> 5;
                    for (int i = threadIdx.x; i < SNW * nw; i += NT) S.wm[i] = 0u;
                    __syncthreads();
                    soft_stage_group(t, sb, nb, base, S.taus, 1, tc, S.need, S.sid, S.rec, S.wm);
                    __syncthreads();
                    if (mine) soft_product(S.rec, S.wm + warp * nw, nw, ul, vl, kexp, P, Pnz, nz);
                    base += nb;
                    __syncthreads();
                }
                if (mine) { S.pnz[0][myp] = Pnz; S.nz[0][myp] = nz; }
                __syncthreads();
                base = 0;
                fpos = 0;
                while (true) {   // pass 2: re-stage each batch
                    const int nb = sb.fb ? soft_fallback_fill(t, sb.rseg, S.taus[0], tc, SREC_S, fpos, S.sid, S.wsum)
                                         : (base < sb.n ? min(SREC_S, sb.n - base) : 0);
                    if (nb == 0) break;
                    const int nw = (nb + 31) >> 5;
                    for (int i = threadIdx.x; i < SNW * nw; i += NT) S.wm[i] = 0u;
                    __syncthreads();
                    soft_stage_group(t, sb, nb, base, S.taus, 1, tc, S.need, S.sid, S.rec, S.wm);
                    __syncthreads();
                    soft_grad_group(S, t, im, ch.s, nb, 1, tc, sb.fb ? 0 : base, false, acc0, acc1,
                                    sb.fb ? S.sid : sb.ent);
                    base += nb;
                    __syncthreads();
                }
            }
        }
    }
}

}  // namespace

cudaError_t launch_soft_fwd(const Tables &t, float *out, cudaStream_t st)
{
    if (t.B == 0 || t.T == 0) return cudaSuccess;
    const size_t n = (size_t)t.B * t.H * t.W;
    cudaError_t e;
    if (t.F > 0) {
        const int smem = (int)sizeof(SoftFwdSmem);
        e = cudaFuncSetAttribute(k8_soft_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        k8_soft_fwd<<<dim3(t.T, t.B, t.splits), NT, smem, st>>>(t);
    } else {
        e = cudaMemsetAsync(t.spart, 0, sizeof(float) * n * t.splits, st);
        if (e != cudaSuccess) return e;
    }
    const unsigned blocks = (unsigned)std::min<size_t>((n + 255) / 256, 148 * 16);
    k8_soft_reduce<<<blocks, 256, 0, st>>>(t.spart, reinterpret_cast<float4 *>(out), n, t.splits);
    return cudaGetLastError();
}

cudaError_t launch_soft_bwd(const Tables &t, const float *grad, cudaStream_t st)
{
    if (t.B == 0 || t.T == 0 || t.F == 0) return cudaSuccess;
    const int smem = (int)sizeof(SoftBwdSmem);
    cudaError_t e = cudaFuncSetAttribute(k9_soft_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    k9_soft_bwd<<<dim3(t.T, t.B, t.splits), NT, smem, st>>>(t, grad);
    return cudaGetLastError();
}

}  // namespace br
