// raster_common.cuh -- device helpers shared by the raster kernels (k_raster.cu: the footprint-mask
// generation used by the naive solvers of the NEXT-2 ablation; k_span.cu: the span raster of the
// fast solver).  Not part of the ABI.
#pragma once
#include "internal.cuh"

namespace br {

constexpr int NWARP = NT / 32;

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

struct FaceRec {            // a (face, segment) coefficient record held in registers
    float4 q[REC_F4];
};

__device__ __forceinline__ void load_rec(const float4 *__restrict__ r, FaceRec &fr)
{
#pragma unroll
    for (int i = 0; i < REC_F4; ++i) fr.q[i] = __ldg(r + i);
}

// Fallback batch builder: faces whose per-tau box overlaps the tile, in index order, from fpos on.
// Block-uniform.  Returns the batch size (0 when all faces are consumed).
static __device__ int fallback_fill(const float4 *__restrict__ rseg, int F, float tau, const TileCtx &tc, int W, int H,
                             int cap, int &fpos, int *sid, int *swsum)
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
        for (int w = 0; w < NWARP; ++w) {
            const int c = swsum[w];
            pre += w < warp ? c : 0;
            tot += c;
        }
        __syncthreads();
        if (nb + tot > cap) break;                       // uniform: batch full
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
    const float4 *key0;   // keyframes s and s+1 of the image (naive solvers, NEXT-2)
    const float4 *key1;
    const float4 *fcol;
    const int *ent;       // sorted bin entries (normal path)
    int n;                // bin length
    bool fb;              // fallback path
};

// Per-sub-frame batch iteration (bins longer than the record capacity, fallback): returns nb
// (0 = done).  Normal path: contiguous slices of the sorted bin.  Fallback: faces rescanned.
__device__ __forceinline__ int next_batch(const BinCtx &bc, int F, float tau, const TileCtx &tc, int W, int H,
                                          int cap, int base, int &fpos, int *sid, int *swsum)
{
    if (!bc.fb) return base < bc.n ? min(cap, bc.n - base) : 0;
    return fallback_fill(bc.rseg, F, tau, tc, W, H, cap, fpos, sid, swsum);
}

template <class R>
__device__ __forceinline__ void weights(const R &r, float ul, float vl, float w[3])
{
    w[0] = edge_eval(r.a[0], r.b[0], r.g[0], ul, vl) * r.invD;
    w[1] = edge_eval(r.a[1], r.b[1], r.g[1], ul, vl) * r.invD;
    w[2] = edge_eval(r.a[2], r.b[2], r.g[2], ul, vl) * r.invD;
}

template <class R>
__device__ __forceinline__ void shade(const R &r, const float4 *__restrict__ fcol, float ul, float vl,
                                      float &pr, float &pg, float &pb)
{
    float w[3];
    weights(r, ul, vl, w);
    const float4 *fc = fcol + 3 * (size_t)r.fid;
    const float4 c0 = __ldg(fc), c1 = __ldg(fc + 1), c2 = __ldg(fc + 2);
    pr = __fmaf_rn(w[0], c0.x, __fmaf_rn(w[1], c0.w, w[2] * c1.z));
    pg = __fmaf_rn(w[0], c0.y, __fmaf_rn(w[1], c1.x, w[2] * c1.w));
    pb = __fmaf_rn(w[0], c0.z, __fmaf_rn(w[1], c1.y, w[2] * c2.x));
}

__device__ __forceinline__ void tile_ctx(const Tables &t, int tile, TileCtx &tc)
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

// closed-form face gradient at tau from its moments m = sum over the face's won pixels of
// g (1, u, v) (g = dL/dI_k): dL/dc_i = (A_i mu + B_i mv + G_i m0) / |D|,
// dL/dv_i = -(A_i (PA.mu) + B_i (PA.mv) + G_i (PA.m0), same with PB) / D^2, PA = sum_j A_j c_j,
// PB = sum_j B_j c_j (Eq.9 and dw/dv_i = -w_i dw/dp; k_raster.cu / k_span.cu backward comments)
template <class R>
__device__ __forceinline__ void face_grad(const R &r, const float m[9], const float4 *__restrict__ fcol,
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

}  // namespace br
