// k_optim.cu -- NEXT-4: the kernels of a translational recovery iteration besides the renderer
// (include/blurrast_optim.h): L1 image loss (Eq.16), Laplacian (A21) and smoothness (A22)
// regularisers, Adam, and the evaluation metrics (sum of squared differences for PSNR, voxel IoU).
// All elementwise / per-vertex / per-edge work is HBM-bound and tiny next to the renderer; the
// kernels are grid-stride loops sized to the SM count, with warp-shuffle + one atomic per warp for
// the loss scalars.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "internal.cuh"
#include "../../include/blurrast_optim.h"

namespace br {

namespace {


__device__ __forceinline__ float warp_sum(float x)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

__device__ __forceinline__ double warp_sum_d(double x)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

__device__ __forceinline__ float sgnf(float x) { return x > 0.f ? 1.f : (x < 0.f ? -1.f : 0.f); }

// ---- L1 image loss (Eq.16): one float4 (pixel) per iteration
__global__ void __launch_bounds__(256) k_l1(const float4 *__restrict__ o, const float4 *__restrict__ t, long long npix,
                                            long long hw, const uint8_t *__restrict__ mask, float irgb, float ia,
                                            float *loss, float4 *__restrict__ g)
{
    float s = 0.f;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < npix;
         i += (long long)gridDim.x * blockDim.x) {
        const bool on = mask == nullptr || mask[i / hw] != 0;
        float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
        if (on) {
            const float4 a = __ldg(o + i), b = __ldg(t + i);
            const float dx = a.x - b.x, dy = a.y - b.y, dz = a.z - b.z, dw = a.w - b.w;
            s += (fabsf(dx) + fabsf(dy) + fabsf(dz)) * irgb + fabsf(dw) * ia;
            r = make_float4(sgnf(dx) * irgb, sgnf(dy) * irgb, sgnf(dz) * irgb, sgnf(dw) * ia);
        }
        g[i] = r;
    }
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0 && s != 0.f) atomicAdd(loss, s);
}

// ---- Laplacian (A21): r_v = delta_v - mean_{N(v)} delta; L = sum |r_v|^2;
// dL/ddelta_u = 2 r_u - sum_{v in N(u)} 2 r_v / |N(v)|   (N symmetric)
struct Topo {
    int V, E, nnz, pad;
    const int *row;     // [V+1]
    const int *col;     // [nnz]
    const int4 *edge;   // [E] (a, b, c, d)
    float *scratch;     // [3V]
};

__host__ __device__ inline size_t topo_int_words(int V, int nnz, int E) { return 4 + (size_t)(V + 1) + nnz + 4 * (size_t)E; }

__device__ __forceinline__ Topo topo_view(void *base)
{
    int *h = reinterpret_cast<int *>(base);
    Topo t;
    t.V = h[0]; t.E = h[1]; t.nnz = h[2];
    t.row = h + 4;
    t.col = t.row + t.V + 1;
    size_t w = topo_int_words(t.V, t.nnz, 0);
    w = (w + 3) & ~(size_t)3;                        // int4 alignment
    t.edge = reinterpret_cast<const int4 *>(h + w);
    t.scratch = reinterpret_cast<float *>(h + w + 4 * (size_t)t.E);
    return t;
}

__global__ void __launch_bounds__(256) k_lap_r(const float *__restrict__ x, const float *__restrict__ x0, void *topo,
                                               float *loss)
{
    const Topo tp = topo_view(topo);
    float s = 0.f;
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < tp.V; v += gridDim.x * blockDim.x) {
        const int r0 = tp.row[v], r1 = tp.row[v + 1];
        float rx = 0.f, ry = 0.f, rz = 0.f;
        if (r1 > r0) {
            float mx = 0.f, my = 0.f, mz = 0.f;
            for (int q = r0; q < r1; ++q) {
                const int u = tp.col[q];
                mx += x[3 * u] - x0[3 * u];
                my += x[3 * u + 1] - x0[3 * u + 1];
                mz += x[3 * u + 2] - x0[3 * u + 2];
            }
            const float inv = 1.0f / (float)(r1 - r0);
            rx = (x[3 * v] - x0[3 * v]) - mx * inv;
            ry = (x[3 * v + 1] - x0[3 * v + 1]) - my * inv;
            rz = (x[3 * v + 2] - x0[3 * v + 2]) - mz * inv;
            s += rx * rx + ry * ry + rz * rz;
        }
        tp.scratch[3 * v] = rx;
        tp.scratch[3 * v + 1] = ry;
        tp.scratch[3 * v + 2] = rz;
    }
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0 && s != 0.f) atomicAdd(loss, s);
}

__global__ void __launch_bounds__(256) k_lap_g(void *topo, float w, float *__restrict__ g)
{
    const Topo tp = topo_view(topo);
    for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < tp.V; u += gridDim.x * blockDim.x) {
        const int r0 = tp.row[u], r1 = tp.row[u + 1];
        if (r1 == r0) continue;
        float gx = 2.f * tp.scratch[3 * u], gy = 2.f * tp.scratch[3 * u + 1], gz = 2.f * tp.scratch[3 * u + 2];
        for (int q = r0; q < r1; ++q) {
            const int v = tp.col[q];
            const float c = 2.f / (float)(tp.row[v + 1] - tp.row[v]);
            gx -= c * tp.scratch[3 * v];
            gy -= c * tp.scratch[3 * v + 1];
            gz -= c * tp.scratch[3 * v + 2];
        }
        g[3 * u] += w * gx;
        g[3 * u + 1] += w * gy;
        g[3 * u + 2] += w * gz;
    }
}

// ---- smoothness (A22): per interior edge (a, b; wings c, d), e = b - a, c' = c - a, d' = d - a,
// al = c'.e/e.e, be = d'.e/e.e, u = c' - al e, w = d' - be e, cos = u.w / (|u||w|);
// dcos/dc = (w^ - cos u^)/|u| = Gc, dcos/dd = (u^ - cos w^)/|w| = Gd, dcos/db = -al Gc - be Gd,
// dcos/da = -(1 - al) Gc - (1 - be) Gd;  L_e = (cos + 1)^2, dL_e = 2 (cos + 1) dcos.
__global__ void __launch_bounds__(256) k_smooth(const float *__restrict__ x, const void *topo, float wgt, float *loss,
                                                float *__restrict__ g)
{
    const Topo tp = topo_view(const_cast<void *>(topo));
    float s = 0.f;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < tp.E; i += gridDim.x * blockDim.x) {
        const int4 q = tp.edge[i];
        const float ax = x[3 * q.x], ay = x[3 * q.x + 1], az = x[3 * q.x + 2];
        const float ex = x[3 * q.y] - ax, ey = x[3 * q.y + 1] - ay, ez = x[3 * q.y + 2] - az;
        const float cx = x[3 * q.z] - ax, cy = x[3 * q.z + 1] - ay, cz = x[3 * q.z + 2] - az;
        const float dx = x[3 * q.w] - ax, dy = x[3 * q.w + 1] - ay, dz = x[3 * q.w + 2] - az;
        const float ee = ex * ex + ey * ey + ez * ez;
        if (!(ee > 0.f)) continue;
        const float al = (cx * ex + cy * ey + cz * ez) / ee, be = (dx * ex + dy * ey + dz * ez) / ee;
        const float ux = cx - al * ex, uy = cy - al * ey, uz = cz - al * ez;
        const float wx = dx - be * ex, wy = dy - be * ey, wz = dz - be * ez;
        const float nu2 = ux * ux + uy * uy + uz * uz, nw2 = wx * wx + wy * wy + wz * wz;
        if (!(nu2 > 0.f) || !(nw2 > 0.f)) continue;
        const float nu = sqrtf(nu2), nw = sqrtf(nw2);
        const float cs = (ux * wx + uy * wy + uz * wz) / (nu * nw);
        s += (cs + 1.f) * (cs + 1.f);
        const float k = wgt * 2.f * (cs + 1.f);
        const float iu = 1.f / nu, iw = 1.f / nw;
        // Gc = (w^ - cos u^)/|u|, Gd = (u^ - cos w^)/|w|
        const float gcx = (wx * iw - cs * ux * iu) * iu, gcy = (wy * iw - cs * uy * iu) * iu,
                    gcz = (wz * iw - cs * uz * iu) * iu;
        const float gdx = (ux * iu - cs * wx * iw) * iw, gdy = (uy * iu - cs * wy * iw) * iw,
                    gdz = (uz * iu - cs * wz * iw) * iw;
        atomicAdd(g + 3 * q.z, k * gcx);
        atomicAdd(g + 3 * q.z + 1, k * gcy);
        atomicAdd(g + 3 * q.z + 2, k * gcz);
        atomicAdd(g + 3 * q.w, k * gdx);
        atomicAdd(g + 3 * q.w + 1, k * gdy);
        atomicAdd(g + 3 * q.w + 2, k * gdz);
        atomicAdd(g + 3 * q.y, -k * (al * gcx + be * gdx));
        atomicAdd(g + 3 * q.y + 1, -k * (al * gcy + be * gdy));
        atomicAdd(g + 3 * q.y + 2, -k * (al * gcz + be * gdz));
        atomicAdd(g + 3 * q.x, -k * ((1.f - al) * gcx + (1.f - be) * gdx));
        atomicAdd(g + 3 * q.x + 1, -k * ((1.f - al) * gcy + (1.f - be) * gdy));
        atomicAdd(g + 3 * q.x + 2, -k * ((1.f - al) * gcz + (1.f - be) * gdz));
    }
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0 && s != 0.f) atomicAdd(loss, s);
}

// ---- Adam
__global__ void __launch_bounds__(256) k_adam(float *__restrict__ p, const float *__restrict__ g, float *__restrict__ m,
                                              float *__restrict__ v, long long n, float lr, float b1, float b2,
                                              float eps, float ibc1, float ibc2)
{
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const float gi = g[i];
        const float mi = b1 * m[i] + (1.f - b1) * gi;
        const float vi = b2 * v[i] + (1.f - b2) * gi * gi;
        m[i] = mi;
        v[i] = vi;
        p[i] -= lr * (mi * ibc1) / (sqrtf(vi * ibc2) + eps);
    }
}

// ---- sum of squared differences (PSNR)
__global__ void __launch_bounds__(256) k_ssd(const float *__restrict__ a, const float *__restrict__ b, long long n,
                                             double *out)
{
    double s = 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double d = (double)a[i] - (double)b[i];
        s += d * d;
    }
    s = warp_sum_d(s);
    if ((threadIdx.x & 31) == 0 && s != 0.0) atomicAdd(out, s);
}

// ---- voxel IoU: bounding cube (fp64, same operation order as the oracle), ray parity occupancy
struct VoxBox {
    double lo[3], size, h, ny, nz;
};

__global__ void __launch_bounds__(256) k_vox_box(const float *__restrict__ va, int Va, const float *__restrict__ vb,
                                                 int Vb, VoxBox *box)
{
    __shared__ double smn[3][256], smx[3][256];
    double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int i = threadIdx.x; i < Va + Vb; i += blockDim.x) {
        const float *p = i < Va ? va + 3 * i : vb + 3 * (i - Va);
        for (int c = 0; c < 3; ++c) {
            mn[c] = fmin(mn[c], (double)p[c]);
            mx[c] = fmax(mx[c], (double)p[c]);
        }
    }
    for (int c = 0; c < 3; ++c) { smn[c][threadIdx.x] = mn[c]; smx[c][threadIdx.x] = mx[c]; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double lo[3], hi[3];
        for (int c = 0; c < 3; ++c) {
            lo[c] = INFINITY; hi[c] = -INFINITY;
            for (int i = 0; i < (int)blockDim.x; ++i) { lo[c] = fmin(lo[c], smn[c][i]); hi[c] = fmax(hi[c], smx[c][i]); }
        }
        double ext = __dsub_rn(hi[0], lo[0]);
        ext = fmax(ext, __dsub_rn(hi[1], lo[1]));
        ext = fmax(ext, __dsub_rn(hi[2], lo[2]));
        const double size = __dmul_rn(ext, 1.02);
        for (int c = 0; c < 3; ++c) box->lo[c] = __dsub_rn(__dmul_rn(0.5, __dadd_rn(lo[c], hi[c])), __dmul_rn(0.5, size));
        box->size = size;
    }
}

constexpr int VOX_MAXHIT = 256;

// one thread per (j, k) ray; occ[(i * res + j) * res + k]
__global__ void __launch_bounds__(128) k_vox_occ(const float *__restrict__ v, const int *__restrict__ f, int F,
                                                 const VoxBox *box, int res, uint8_t *__restrict__ occ, int *ovf)
{
    const int jk = blockIdx.x * blockDim.x + threadIdx.x;
    if (jk >= res * res) return;
    const int j = jk / res, k = jk - j * res;
    const double size = box->size, h = size / (double)res;
    const double y = __dadd_rn(__dadd_rn(box->lo[1], __dmul_rn((double)j + 0.5, h)), __dmul_rn(__dmul_rn(1e-7, sqrt(2.0)), h));
    const double z = __dadd_rn(__dadd_rn(box->lo[2], __dmul_rn((double)k + 0.5, h)), __dmul_rn(__dmul_rn(1e-7, sqrt(3.0)), h));
    double hits[VOX_MAXHIT];
    int nh = 0;
    for (int q = 0; q < F; ++q) {
        const int a = f[3 * q], b = f[3 * q + 1], c = f[3 * q + 2];
        const double y0 = v[3 * a + 1], z0 = v[3 * a + 2], y1 = v[3 * b + 1], z1 = v[3 * b + 2];
        const double y2 = v[3 * c + 1], z2 = v[3 * c + 2];
        const double s0 = __dsub_rn(__dmul_rn(__dsub_rn(y1, y), __dsub_rn(z2, z)), __dmul_rn(__dsub_rn(y2, y), __dsub_rn(z1, z)));
        const double s1 = __dsub_rn(__dmul_rn(__dsub_rn(y2, y), __dsub_rn(z0, z)), __dmul_rn(__dsub_rn(y0, y), __dsub_rn(z2, z)));
        const double s2 = __dsub_rn(__dmul_rn(__dsub_rn(y0, y), __dsub_rn(z1, z)), __dmul_rn(__dsub_rn(y1, y), __dsub_rn(z0, z)));
        const bool in = (s0 > 0 && s1 > 0 && s2 > 0) || (s0 < 0 && s1 < 0 && s2 < 0);
        if (!in) continue;
        const double den = __dadd_rn(__dadd_rn(s0, s1), s2);
        const double num = __dadd_rn(__dadd_rn(__dmul_rn(s0, (double)v[3 * a]), __dmul_rn(s1, (double)v[3 * b])),
                                     __dmul_rn(s2, (double)v[3 * c]));
        if (nh < VOX_MAXHIT) hits[nh++] = __ddiv_rn(num, den);
        else *ovf = 1;
    }
    for (int i = 0; i < res; ++i) {
        const double x = __dadd_rn(box->lo[0], __dmul_rn((double)i + 0.5, h));
        int cnt = 0;
        for (int q = 0; q < nh; ++q) cnt += hits[q] > x;
        occ[((size_t)i * res + j) * res + k] = (uint8_t)(cnt & 1);
    }
}

__global__ void __launch_bounds__(256) k_vox_count(const uint8_t *__restrict__ a, const uint8_t *__restrict__ b, int n,
                                                   unsigned long long *counts)
{
    unsigned long long in = 0, un = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        in += a[i] & b[i];
        un += a[i] | b[i];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        in += __shfl_xor_sync(0xffffffffu, in, o);
        un += __shfl_xor_sync(0xffffffffu, un, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (in) atomicAdd(counts, in);
        if (un) atomicAdd(counts + 1, un);
    }
}

int ofail(int code, const std::string &m)
{
    set_last_error(m);   // reported by blur_last_error() (abi.cu)
    return code;
}

int ocheck(cudaError_t e, const char *what)
{
    if (e != cudaSuccess) return ofail(BLUR_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
    return BLUR_OK;
}

unsigned grid_for(long long n, int per = 256)
{
    const long long b = (n + per - 1) / per;
    return (unsigned)std::max(1LL, std::min(b, 148LL * 8));
}

struct HostTopo {
    std::vector<int> row, col;
    std::vector<int> edge;   // 4 per interior edge
};

bool build_host_topo(int V, int F, const int32_t *faces, HostTopo &h)
{
    std::vector<std::vector<int>> nb((size_t)V);
    std::vector<std::array<int, 3>> ek;   // (min, max, opposite)
    ek.reserve((size_t)3 * F);
    for (int q = 0; q < F; ++q) {
        for (int i = 0; i < 3; ++i) {
            const int a = faces[3 * q + i], b = faces[3 * q + (i + 1) % 3], c = faces[3 * q + (i + 2) % 3];
            if (a < 0 || a >= V || b < 0 || b >= V || c < 0 || c >= V) return false;
            if (a != b) {
                nb[a].push_back(b);
                nb[b].push_back(a);
            }
            ek.push_back({std::min(a, b), std::max(a, b), c});
        }
    }
    h.row.assign((size_t)V + 1, 0);
    for (int v = 0; v < V; ++v) {
        std::sort(nb[v].begin(), nb[v].end());
        nb[v].erase(std::unique(nb[v].begin(), nb[v].end()), nb[v].end());
        h.row[v + 1] = h.row[v] + (int)nb[v].size();
    }
    h.col.reserve(h.row[V]);
    for (int v = 0; v < V; ++v) h.col.insert(h.col.end(), nb[v].begin(), nb[v].end());
    std::sort(ek.begin(), ek.end());
    for (size_t i = 0; i < ek.size();) {
        size_t j = i + 1;
        while (j < ek.size() && ek[j][0] == ek[i][0] && ek[j][1] == ek[i][1]) ++j;
        if (j - i == 2 && ek[i][0] != ek[i][1]) {
            h.edge.push_back(ek[i][0]);
            h.edge.push_back(ek[i][1]);
            h.edge.push_back(ek[i][2]);
            h.edge.push_back(ek[i + 1][2]);
        }
        i = j;
    }
    return true;
}

size_t topo_bytes_of(int V, const HostTopo &h)
{
    const int E = (int)h.edge.size() / 4;
    size_t w = topo_int_words(V, (int)h.col.size(), 0);
    w = (w + 3) & ~(size_t)3;
    return 4 * (w + 4 * (size_t)E) + 4 * 3 * (size_t)V;
}

}  // namespace

}  // namespace br

using namespace br;

extern "C" {

size_t blur_topology_bytes(int V, int F, const int32_t *faces_host)
{
    clear_last_error();
    if (V < 0 || F < 0 || (F > 0 && !faces_host)) { ofail(BLUR_EINVAL, "bad topology arguments"); return 0; }
    HostTopo h;
    if (!build_host_topo(V, F, faces_host, h)) { ofail(BLUR_EINVAL, "face index out of range [0, V)"); return 0; }
    return topo_bytes_of(V, h);
}

int blur_topology_build(int V, int F, const int32_t *faces_host, void *topo, size_t topo_bytes, blur_stream_t stream)
{
    clear_last_error();
    if (V < 0 || F < 0 || (F > 0 && !faces_host) || !topo) return ofail(BLUR_EINVAL, "bad topology arguments");
    HostTopo h;
    if (!build_host_topo(V, F, faces_host, h)) return ofail(BLUR_EINVAL, "face index out of range [0, V)");
    const size_t need = topo_bytes_of(V, h);
    if (topo_bytes < need) return ofail(BLUR_ENOMEM, "topology buffer too small: need " + std::to_string(need));
    const int E = (int)h.edge.size() / 4, nnz = (int)h.col.size();
    size_t w = topo_int_words(V, nnz, 0);
    w = (w + 3) & ~(size_t)3;
    std::vector<int> buf(w + 4 * (size_t)E, 0);
    buf[0] = V; buf[1] = E; buf[2] = nnz;
    std::memcpy(buf.data() + 4, h.row.data(), sizeof(int) * h.row.size());
    if (nnz) std::memcpy(buf.data() + 4 + V + 1, h.col.data(), sizeof(int) * nnz);
    if (E) std::memcpy(buf.data() + w, h.edge.data(), sizeof(int) * h.edge.size());
    cudaStream_t st = (cudaStream_t)stream;
    int r = ocheck(cudaMemcpyAsync(topo, buf.data(), sizeof(int) * buf.size(), cudaMemcpyHostToDevice, st), "topology copy");
    if (r) return r;
    return ocheck(cudaStreamSynchronize(st), "topology sync");
}

int blur_l1_loss_grad(const float *out, const float *target, int B, int H, int W, const uint8_t *image_mask,
                      int n_images, float *loss, float *grad, blur_stream_t stream)
{
    clear_last_error();
    if (B < 0 || H < 1 || W < 1 || !loss) return ofail(BLUR_EINVAL, "bad L1 arguments");
    if (B > 0 && (!out || !target || !grad)) return ofail(BLUR_EINVAL, "NULL image pointer");
    if ((((uintptr_t)out) | ((uintptr_t)target) | ((uintptr_t)grad)) & 15)
        return ofail(BLUR_EINVAL, "out/target/grad must be 16-byte aligned");
    if (!image_mask) n_images = B;
    if (n_images < 0 || n_images > B) return ofail(BLUR_EINVAL, "n_images not in [0, B]");
    cudaStream_t st = (cudaStream_t)stream;
    int r = ocheck(cudaMemsetAsync(loss, 0, sizeof(float), st), "loss clear");
    if (r || B == 0) return r;
    const long long hw = (long long)H * W, npix = hw * B;
    const double n = (double)n_images * (double)hw;
    const float irgb = n > 0 ? (float)(1.0 / (3.0 * n)) : 0.f, ia = n > 0 ? (float)(1.0 / n) : 0.f;
    k_l1<<<grid_for(npix), 256, 0, st>>>(reinterpret_cast<const float4 *>(out), reinterpret_cast<const float4 *>(target),
                                         npix, hw, image_mask, irgb, ia, loss, reinterpret_cast<float4 *>(grad));
    return ocheck(cudaGetLastError(), "l1 kernel");
}

int blur_laplacian_loss_grad(const float *verts, const float *verts0, int V, void *topo, float weight, float *loss,
                             float *grad_verts, blur_stream_t stream)
{
    clear_last_error();
    if (V < 0 || !topo || !loss || (V > 0 && (!verts || !verts0 || !grad_verts)))
        return ofail(BLUR_EINVAL, "bad Laplacian arguments");
    cudaStream_t st = (cudaStream_t)stream;
    int r = ocheck(cudaMemsetAsync(loss, 0, sizeof(float), st), "loss clear");
    if (r || V == 0) return r;
    k_lap_r<<<grid_for(V), 256, 0, st>>>(verts, verts0, topo, loss);
    k_lap_g<<<grid_for(V), 256, 0, st>>>(topo, weight, grad_verts);
    return ocheck(cudaGetLastError(), "laplacian kernels");
}

int blur_smooth_loss_grad(const float *verts, int V, const void *topo, float weight, float *loss, float *grad_verts,
                          blur_stream_t stream)
{
    clear_last_error();
    if (V < 0 || !topo || !loss || (V > 0 && (!verts || !grad_verts))) return ofail(BLUR_EINVAL, "bad smoothness arguments");
    cudaStream_t st = (cudaStream_t)stream;
    int r = ocheck(cudaMemsetAsync(loss, 0, sizeof(float), st), "loss clear");
    if (r || V == 0) return r;
    k_smooth<<<148 * 4, 256, 0, st>>>(verts, topo, weight, loss, grad_verts);
    return ocheck(cudaGetLastError(), "smoothness kernel");
}

int blur_adam_step(float *params, const float *grads, float *m, float *v, int64_t n, int step, float lr, float beta1,
                   float beta2, float eps, blur_stream_t stream)
{
    clear_last_error();
    if (n < 0 || step < 1 || (n > 0 && (!params || !grads || !m || !v))) return ofail(BLUR_EINVAL, "bad Adam arguments");
    if (!(beta1 >= 0.f && beta1 < 1.f && beta2 >= 0.f && beta2 < 1.f)) return ofail(BLUR_EINVAL, "betas not in [0, 1)");
    if (n == 0) return BLUR_OK;
    const double bc1 = 1.0 - std::pow((double)beta1, step), bc2 = 1.0 - std::pow((double)beta2, step);
    k_adam<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(params, grads, m, v, n, lr, beta1, beta2, eps,
                                                          (float)(1.0 / bc1), (float)(1.0 / bc2));
    return ocheck(cudaGetLastError(), "adam kernel");
}

int blur_sum_sq_diff(const float *a, const float *b, int64_t n, double *sum_sq, blur_stream_t stream)
{
    clear_last_error();
    if (n < 0 || !sum_sq || (n > 0 && (!a || !b))) return ofail(BLUR_EINVAL, "bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    int r = ocheck(cudaMemsetAsync(sum_sq, 0, sizeof(double), st), "clear");
    if (r || n == 0) return r;
    k_ssd<<<grid_for(n), 256, 0, st>>>(a, b, n, sum_sq);
    return ocheck(cudaGetLastError(), "ssd kernel");
}

size_t blur_voxel_scratch_bytes(int res)
{
    if (res < 2 || res > 512) return 0;
    return 256 + 2 * (size_t)res * res * res + 16;
}

int blur_voxel_iou(const float *va, int Va, const int32_t *fa, int Fa, const float *vb, int Vb, const int32_t *fb,
                   int Fb, int res, void *scratch, size_t scratch_bytes, unsigned long long *counts,
                   blur_stream_t stream)
{
    clear_last_error();
    if (res < 2 || res > 512) return ofail(BLUR_EINVAL, "res must be in [2, 512]");
    if (Va < 1 || Vb < 1 || Fa < 0 || Fb < 0 || !va || !vb || !counts || (Fa && !fa) || (Fb && !fb))
        return ofail(BLUR_EINVAL, "bad mesh arguments");
    if (!scratch || scratch_bytes < blur_voxel_scratch_bytes(res)) return ofail(BLUR_ENOMEM, "voxel scratch too small");
    cudaStream_t st = (cudaStream_t)stream;
    char *s = (char *)scratch;
    VoxBox *box = reinterpret_cast<VoxBox *>(s);
    uint8_t *oa = reinterpret_cast<uint8_t *>(s + 256), *ob = oa + (size_t)res * res * res;
    int *ovf = reinterpret_cast<int *>(ob + (size_t)res * res * res);
    int r = ocheck(cudaMemsetAsync(counts, 0, 16, st), "clear");
    if (r) return r;
    r = ocheck(cudaMemsetAsync(ovf, 0, sizeof(int), st), "clear");
    if (r) return r;
    k_vox_box<<<1, 256, 0, st>>>(va, Va, vb, Vb, box);
    const unsigned g = (unsigned)((res * res + 127) / 128);
    k_vox_occ<<<g, 128, 0, st>>>(va, fa, Fa, box, res, oa, ovf);
    k_vox_occ<<<g, 128, 0, st>>>(vb, fb, Fb, box, res, ob, ovf);
    k_vox_count<<<grid_for((long long)res * res * res), 256, 0, st>>>(oa, ob, res * res * res, counts);
    return ocheck(cudaGetLastError(), "voxel kernels");
}

}  // extern "C"
