// k_setup.cu -- K1 (keyframe pose + projection) and K2 (per-segment fast-solver coefficients).
//
// K1  one thread per (image b, keyframe s, vertex v): exact rigid pose at t = s/S (A30/A31
//     generalised, Q2-Q4), view transform and perspective projection A34, in fp64,
//     rounded once to fp32.  Output float4 (x_ndc, y_ndc, z_view, valid).
// K2  one thread per (image b, segment s, face f): "the coefficients (A1, A2, A3, a1, a2, a3) can
//     be computed only once".  The numerator of w_i (Eq.7-8) is the edge function of the
//     edge opposite corner i; it is formed from keyframe edge vectors (e0 = b - a, de, da) about the
//     edge's canonical start vertex a (lower vertex index), so the two faces sharing an edge store
//     bit-identical coefficients up to sign (watertight coverage).  det F(tau) = d3 + tau(d2 + tau d1)
//     from keyframe edge vectors (A8 regrouped).  The A11-A16 expansion itself is ill-conditioned
//     in fp32; this is the same polynomial, see DESIGN.md.
#include <algorithm>

#include "internal.cuh"
#include "../../include/blurrast.h"

namespace br {

__global__ void __launch_bounds__(256) k1_keyframes(Tables t, const float *__restrict__ verts)
{
    const int b = blockIdx.y;
    const ImgInfo &im = t.imgs[b];
    const int V = t.V;
    const int nk = (im.S + 1) * V;
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx == 0 && b == 0) {
        *t.orient = 0.0;                  // K2 accumulates the mesh orientation after this kernel
        if (t.vg_count) *t.vg_count = 0;  // the visibility gather's leftover list (k_gather.cu) starts empty
    }
    if (idx >= nk) return;
    const int s = idx / V, v = idx - s * V;
    const PoseRec &pr = t.poses[im.pose_off + s];
    const double q[3] = {(double)verts[3 * v] - pr.c[0], (double)verts[3 * v + 1] - pr.c[1],
                         (double)verts[3 * v + 2] - pr.c[2]};
    double P[3], d[3], Q[3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
        P[i] = pr.R[3 * i] * q[0] + pr.R[3 * i + 1] * q[1] + pr.R[3 * i + 2] * q[2] + pr.c[i] + pr.T[i];
#pragma unroll
    for (int i = 0; i < 3; ++i) d[i] = P[i] - im.eye[i];
#pragma unroll
    for (int i = 0; i < 3; ++i) Q[i] = im.Rc[3 * i] * d[0] + im.Rc[3 * i + 1] * d[1] + im.Rc[3 * i + 2] * d[2];
    const bool valid = Q[2] > im.z_near;
    const double den = Q[2] * im.tan_half;
    float4 o;
    o.x = (float)(Q[0] / den);
    o.y = (float)(Q[1] / den);
    o.z = (float)Q[2];
    o.w = valid ? 1.f : 0.f;
    t.key[im.key_off + idx] = o;
    if (!valid) atomicOr(t.status, BLUR_ST_EBEHIND);
}

// explicit-rounding fp64 cross product a x b = ax by - ay bx (same instruction sequence at every
// call site, so shared edges produce identical bits)
__device__ __forceinline__ double xcross(double ax, double ay, double bx, double by)
{
    return __fma_rn(ax, by, -__dmul_rn(ay, bx));
}

// One (image, segment, face) record into out[0..REC_F4) (registers); skipped faces get q6.w = -1.
__device__ __forceinline__ void face_setup(const Tables &t, const ImgInfo &im, int b, int s, int f,
                                           const int *__restrict__ faces, const float *__restrict__ colors,
                                           float4 *out)
{
    const int V = t.V;
    int vid[3] = {faces[3 * f], faces[3 * f + 1], faces[3 * f + 2]};
    const bool oob = vid[0] < 0 || vid[0] >= V || vid[1] < 0 || vid[1] >= V || vid[2] < 0 || vid[2] >= V;
    if (b == 0 && s == 0) {   // per-face colour/index table (image independent)
        float c[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
        if (!oob)
            for (int i = 0; i < 3; ++i)
                for (int ch = 0; ch < 3; ++ch) c[3 * i + ch] = colors[3 * vid[i] + ch];
        float4 *fc = t.fcol + 3 * (size_t)f;
        fc[0] = make_float4(c[0], c[1], c[2], c[3]);
        fc[1] = make_float4(c[4], c[5], c[6], c[7]);
        fc[2] = make_float4(c[8], __int_as_float(oob ? 0 : vid[0]), __int_as_float(oob ? 0 : vid[1]),
                            __int_as_float(oob ? 0 : vid[2]));
    }
    if (oob) {
        if (s == 0) atomicOr(t.status, BLUR_ST_EINVAL);
        out[6] = make_float4(0.f, 0.f, 0.f, __int_as_float(-1));
        return;
    }
    const float4 *k0 = t.key + im.key_off + (size_t)s * V;
    const float4 *k1 = k0 + V;
    float4 p0[3], p1[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) { p0[i] = k0[vid[i]]; p1[i] = k1[vid[i]]; }
    const bool degen = vid[0] == vid[1] || vid[1] == vid[2] || vid[0] == vid[2];
    const bool behind = p0[0].w == 0.f || p0[1].w == 0.f || p0[2].w == 0.f || p1[0].w == 0.f ||
                        p1[1].w == 0.f || p1[2].w == 0.f;
    if (degen || behind) {
        out[6] = make_float4(0.f, 0.f, 0.f, __int_as_float(-1));
        return;
    }
    double X0[3], Y0[3], X1[3], Y1[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) { X0[i] = p0[i].x; Y0[i] = p0[i].y; X1[i] = p1[i].x; Y1[i] = p1[i].y; }
    float e[24];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const int j = (i + 1) % 3, l = (i + 2) % 3;      // N_i = cross(v_l - v_j, p - v_j)
        const bool fwd = vid[j] < vid[l];
        const int a = fwd ? j : l, c = fwd ? l : j;      // canonical edge a -> c
        const float sg = fwd ? 1.f : -1.f;
        const double e0x = __dsub_rn(X0[c], X0[a]), e0y = __dsub_rn(Y0[c], Y0[a]);
        const double e1x = __dsub_rn(X1[c], X1[a]), e1y = __dsub_rn(Y1[c], Y1[a]);
        const double dex = __dsub_rn(e1x, e0x), dey = __dsub_rn(e1y, e0y);
        const double dax = __dsub_rn(X1[a], X0[a]), day = __dsub_rn(Y1[a], Y0[a]);
        e[8 * i + 0] = (float)X0[a];
        e[8 * i + 1] = (float)Y0[a];
        e[8 * i + 2] = sg * (float)(-e0y);                   // a0 = d N / d u at tau = 0
        e[8 * i + 3] = sg * (float)(-dey);                   // a1
        e[8 * i + 4] = sg * (float)e0x;                      // b0 = d N / d v at tau = 0
        e[8 * i + 5] = sg * (float)dex;                      // b1
        e[8 * i + 6] = (float)dax;                          // motion of the canonical vertex over the segment
        e[8 * i + 7] = (float)day;                          // (a position: not sign-flipped)
    }
    // det F(tau) = cross(E1(tau), E2(tau)), E1 = v1 - v0, E2 = v2 - v0 (A8)
    const double E1x = X0[1] - X0[0], E1y = Y0[1] - Y0[0], E2x = X0[2] - X0[0], E2y = Y0[2] - Y0[0];
    const double F1x = X1[1] - X1[0], F1y = Y1[1] - Y1[0], F2x = X1[2] - X1[0], F2y = Y1[2] - Y1[0];
    const double dE1x = F1x - E1x, dE1y = F1y - E1y, dE2x = F2x - E2x, dE2y = F2y - E2y;
    const double d3 = xcross(E1x, E1y, E2x, E2y);
    const double d2 = xcross(E1x, E1y, dE2x, dE2y) + xcross(dE1x, dE1y, E2x, E2y);
    const double d1 = xcross(dE1x, dE1y, dE2x, dE2y);
#pragma unroll
    for (int q = 0; q < 6; ++q) out[q] = make_float4(e[4 * q], e[4 * q + 1], e[4 * q + 2], e[4 * q + 3]);
    out[6] = make_float4((float)d1, (float)d2, (float)d3, __int_as_float(f));
    out[7] = make_float4(fminf(fminf(p0[0].x, p0[1].x), p0[2].x) - BBOX_PAD,
                         fmaxf(fmaxf(p0[0].x, p0[1].x), p0[2].x) + BBOX_PAD,
                         fminf(fminf(p0[0].y, p0[1].y), p0[2].y) - BBOX_PAD,
                         fmaxf(fmaxf(p0[0].y, p0[1].y), p0[2].y) + BBOX_PAD);
    out[8] = make_float4(fminf(fminf(p1[0].x, p1[1].x), p1[2].x) - BBOX_PAD,
                         fmaxf(fmaxf(p1[0].x, p1[1].x), p1[2].x) + BBOX_PAD,
                         fminf(fminf(p1[0].y, p1[1].y), p1[2].y) - BBOX_PAD,
                         fmaxf(fmaxf(p1[0].y, p1[1].y), p1[2].y) + BBOX_PAD);
    out[9] = make_float4(p0[0].z, p0[1].z, p0[2].z, 0.f);
    out[10] = make_float4(p1[0].z, p1[1].z, p1[2].z, 0.f);
}

// K2: thread per (segment, face) of image blockIdx.y; each warp stages its 32 consecutive records in
// shared memory and stores them as one contiguous run (coalesced, instead of 176-B strided stores)
__global__ void __launch_bounds__(256) k2_face_setup(Tables t, const int *__restrict__ faces,
                                                     const float *__restrict__ colors, const float *__restrict__ verts)
{
    __shared__ float4 st[8][32 * REC_F4];
    const int b = blockIdx.y;
    const ImgInfo &im = t.imgs[b];
    const int F = t.F, n = im.S * F;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int base = blockIdx.x * blockDim.x + warp * 32, idx = base + lane;
    if (base >= n) return;   // warp-uniform
    if (b == 0 && base < F) {
        // mesh orientation for the forward's visiting order (k4l_raster_fwd: faces turned towards the camera
        // first, so that the others can be skipped per warp footprint once every pixel there has a nearer
        // winner): sum over faces of det(P0[v0], P0[v1], P0[v2]) = 6 x the signed volume.  Only its sign is
        // used, and only for speed: the raster's result does not depend on it.
        double d = 0.0;
        if (idx < F) {
            const int a = faces[3 * idx], c1 = faces[3 * idx + 1], c2 = faces[3 * idx + 2];
            if ((unsigned)a < (unsigned)t.V && (unsigned)c1 < (unsigned)t.V && (unsigned)c2 < (unsigned)t.V) {
                const double ax = verts[3 * a], ay = verts[3 * a + 1], az = verts[3 * a + 2];
                const double bx = verts[3 * c1], by = verts[3 * c1 + 1], bz = verts[3 * c1 + 2];
                const double cx = verts[3 * c2], cy = verts[3 * c2 + 1], cz = verts[3 * c2 + 2];
                d = ax * (by * cz - bz * cy) + ay * (bz * cx - bx * cz) + az * (bx * cy - by * cx);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
        if (lane == 0 && d != 0.0) atomicAdd(t.orient, d);
    }
    float4 r[REC_F4];
#pragma unroll
    for (int q = 0; q < REC_F4; ++q) r[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (idx < n) {
        const int s = idx / F, f = idx - s * F;
        face_setup(t, im, b, s, f, faces, colors, r);
    }
#pragma unroll
    for (int q = 0; q < REC_F4; ++q) st[warp][lane * REC_F4 + q] = r[q];
    __syncwarp();
    const int cnt = min(32, n - base) * REC_F4;
    float4 *out = t.rec + (size_t)(im.rec_off + base) * REC_F4;
    for (int k = lane; k < cnt; k += 32) out[k] = st[warp][k];
}

cudaError_t launch_setup(const Tables &t, const float *verts, const int *faces, const float *colors,
                         int maxS, cudaStream_t st)
{
    if (t.B == 0 || t.V == 0) return cudaSuccess;
    {
        long long nk = (long long)(maxS + 1) * t.V;
        dim3 grid((unsigned)((nk + 255) / 256), (unsigned)t.B);
        k1_keyframes<<<grid, 256, 0, st>>>(t, verts);
    }
    if (t.F > 0) {
        long long nf = (long long)maxS * t.F;
        dim3 grid((unsigned)((nf + 255) / 256), (unsigned)t.B);
        k2_face_setup<<<grid, 256, 0, st>>>(t, faces, colors, verts);
    }
    return cudaGetLastError();
}

}  // namespace br
