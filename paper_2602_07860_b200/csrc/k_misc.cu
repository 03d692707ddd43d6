// k_misc.cu -- K5 (L2 loss + upstream gradient), K7 (keyframe -> world vertex chain),
// FFMA throughput probe (roofline denominator).
#include "internal.cuh"
#include "../../include/blurrast.h"

namespace br {

// K7: dL/dP0[v] = sum_b sum_s R_s^T Rc^T J(Q)^T dkey[b][s][v]; A34 Jacobian
// J = [[1/(z ta), 0, -x_ndc/z], [0, 1/(z ta), -y_ndc/z]] (Q = view coords, x_ndc = Qx/(z ta)).
// One warp per vertex: the lanes take the (image, keyframe) terms round-robin in fp64 and a fixed
// shuffle tree sums them (deterministic; C4 has ~120 keyframe terms per vertex, so a thread per
// vertex left most SMs idle).
__global__ void __launch_bounds__(256) k7_vertex_chain(Tables t, float *__restrict__ gv)
{
    // CTA = 32 vertices (lanes, so the dkey / key loads of one (image, keyframe) are coalesced) x 8 warps
    // sharing the (image, keyframe) terms round-robin; the warps' fp64 partials are summed in a fixed
    // order (deterministic)
    __shared__ double part[8][3][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int v = blockIdx.x * 32 + lane;
    if (blockIdx.x == 0 && threadIdx.x == 0 && t.vg_count) *t.vg_count = 0;   // the gather's list, for the next backward
    double acc[3] = {0.0, 0.0, 0.0};
    if (v < t.V) {
        int q = 0;   // running index of the (image, keyframe) term
        for (int b = 0; b < t.B; ++b) {
            const ImgInfo &im = t.imgs[b];
            const double itan = 1.0 / im.tan_half;
            for (int s = 0; s <= im.S; ++s, ++q) {
                if ((q & 7) != warp) continue;
                const size_t o = (size_t)im.key_off + (size_t)s * t.V + v;
                const float2 g = t.dkey[o];
                if (g.x == 0.f && g.y == 0.f) continue;
                const float4 kq = t.key[o];
                const double rz = 1.0 / (double)kq.z, iz = rz * itan;
                const double dQ[3] = {g.x * iz, g.y * iz, -((double)g.x * kq.x + (double)g.y * kq.y) * rz};
                double dP[3];
#pragma unroll
                for (int i = 0; i < 3; ++i) dP[i] = im.Rc[i] * dQ[0] + im.Rc[3 + i] * dQ[1] + im.Rc[6 + i] * dQ[2];
                const PoseRec &pr = t.poses[im.pose_off + s];
#pragma unroll
                for (int i = 0; i < 3; ++i) acc[i] += pr.R[i] * dP[0] + pr.R[3 + i] * dP[1] + pr.R[6 + i] * dP[2];
            }
        }
    }
#pragma unroll
    for (int i = 0; i < 3; ++i) part[warp][i][lane] = acc[i];
    __syncthreads();
    if (warp < 3 && v < t.V) {   // warp i sums component i over the 8 warps in order
        double a = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) a += part[w][warp][lane];
        gv[3 * v + warp] = (float)a;
    }
}

cudaError_t launch_vertex_chain(const Tables &t, float *gv, cudaStream_t st)
{
    if (t.V == 0) return cudaSuccess;
    k7_vertex_chain<<<(t.V + 31) / 32, 256, 0, st>>>(t, gv);
    return cudaGetLastError();
}

// K5: loss = sum (o - g)^2 / n_norm, grad = 2 (o - g) / n_norm.  Grid-stride, float4 body.
__global__ void __launch_bounds__(256) k5_l2(const float *__restrict__ o, const float *__restrict__ g, long long n,
                                             float scale, float *loss, float *grad)
{
    float s = 0.f;
    const long long n4 = n / 4;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += stride) {
        const float4 a = __ldg(reinterpret_cast<const float4 *>(o) + i);
        const float4 b = __ldg(reinterpret_cast<const float4 *>(g) + i);
        const float4 d = make_float4(a.x - b.x, a.y - b.y, a.z - b.z, a.w - b.w);
        s += d.x * d.x + d.y * d.y + d.z * d.z + d.w * d.w;
        reinterpret_cast<float4 *>(grad)[i] = make_float4(2.f * scale * d.x, 2.f * scale * d.y, 2.f * scale * d.z,
                                                          2.f * scale * d.w);
    }
    for (long long i = 4 * n4 + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride) {
        const float d = o[i] - g[i];
        s += d * d;
        grad[i] = 2.f * scale * d;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    __shared__ float ws[8];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        float tot = 0.f;
        for (int w = 0; w < 8; ++w) tot += ws[w];
        atomicAdd(loss, tot * scale);
    }
}

cudaError_t launch_l2(const float *o, const float *g, long long n, long long n_norm, float *loss, float *grad,
                      cudaStream_t st)
{
    cudaError_t e = cudaMemsetAsync(loss, 0, sizeof(float), st);
    if (e != cudaSuccess || n == 0) return e;
    const float scale = (float)(1.0 / (double)(n_norm > 0 ? n_norm : n));
    long long blocks = (n / 4 + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    if (blocks < 1) blocks = 1;
    k5_l2<<<(unsigned)blocks, 256, 0, st>>>(o, g, n, scale, loss, grad);
    return cudaGetLastError();
}

// FFMA probe: 8 independent chains per thread (enough ILP to saturate the FMA pipes).
__global__ void __launch_bounds__(256) k_ffma(int iters, float *sink)
{
    float a[8];
    const float x = 1.0f + 1e-7f * threadIdx.x, y = 0.999999f;
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = (float)(i + 1) * 1e-3f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 16; ++u)
#pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = __fmaf_rn(a[i], x, y);
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += a[i];
    sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

cudaError_t launch_ffma_probe(int ctas, int iters, float *sink, cudaStream_t st)
{
    k_ffma<<<ctas, 256, 0, st>>>(iters, sink);
    return cudaGetLastError();
}

}  // namespace br
