// k_bin.cu -- K3: tiled binning of faces per (chunk of sub-frames, tile).
//
// A chunk is a run of <= G consecutive sub-frames of one image inside one segment.  Inside a
// segment every vertex moves linearly in screen space (Eq.5-6), so the screen bounding box of a
// face over [tau_min, tau_max] is the union of its boxes at the two ends; with the keyframe boxes
// lerped (a conservative superset of the lerped triangle's box) this gives the swept box exactly
// as the raster kernel evaluates it per sub-frame (monotone fmaf), so the bin is conservative.
//   K3a count  (chunk, face) -> atomic per (chunk, tile) counters
//   K3b scan   exclusive prefix sum of the counters -> bin offsets
//   K3c fill   (chunk, face) -> entries (unordered)
//   K3d sort   soft bins only: bitonic sort of the face ids (one warp per bin up to SORTCAP, one CTA
//              per bin up to 4096), so that the soft product runs in face order (deterministic).
//              The hard bins stay unsorted: the raster z-buffer breaks depth ties by face index (Q7).
// Entries beyond the capacity are left to the raster kernels' exact fallback path (status bit
// BLUR_ST_EOVERFLOW).
#include <algorithm>
#include <cstdio>

#include "internal.cuh"
#include "../../include/blurrast.h"

namespace br {

__device__ __forceinline__ float lerpf_(float tau, float a, float b) { return box_lerp(tau, a, b); }

// NDC box -> inclusive pixel index ranges (Q9 pixel centres); returns false if empty
__device__ __forceinline__ bool ndc_box_to_pixels(float xmn, float xmx, float ymn, float ymx, int W, int H,
                                                  int &i0, int &i1, int &j0, int &j1)
{
    float a, b, c, d;
    ndc_to_index(xmn, xmx, W, false, a, b);
    ndc_to_index(ymn, ymx, H, true, c, d);
    a = fmaxf(a, 0.f);
    b = fminf(b, (float)(W - 1));
    c = fmaxf(c, 0.f);
    d = fminf(d, (float)(H - 1));
    if (!(a <= b) || !(c <= d)) return false;   // also rejects NaN
    i0 = (int)a; i1 = (int)b; j0 = (int)c; j1 = (int)d;
    return true;
}

// swept box of the chunk, grown by dil (soft bins: the NEXT-1 cut-off radius; 0 for the hard bins)
__device__ __forceinline__ bool swept_tiles(const Tables &t, const float4 *r, float tmin, float tmax, float dil,
                                            int &tx0, int &tx1, int &ty0, int &ty1)
{
    const float4 q6 = r[6];
    if (__float_as_int(q6.w) < 0) return false;
    const float4 b0 = r[7], b1 = r[8];
    const float xmn = __fsub_rn(fminf(lerpf_(tmin, b0.x, b1.x), lerpf_(tmax, b0.x, b1.x)), dil);
    const float xmx = __fadd_rn(fmaxf(lerpf_(tmin, b0.y, b1.y), lerpf_(tmax, b0.y, b1.y)), dil);
    const float ymn = __fsub_rn(fminf(lerpf_(tmin, b0.z, b1.z), lerpf_(tmax, b0.z, b1.z)), dil);
    const float ymx = __fadd_rn(fmaxf(lerpf_(tmin, b0.w, b1.w), lerpf_(tmax, b0.w, b1.w)), dil);
    int i0, i1, j0, j1;
    if (!ndc_box_to_pixels(xmn, xmx, ymn, ymx, t.W, t.H, i0, i1, j0, j1)) return false;
    tx0 = i0 / TW; tx1 = i1 / TW; ty0 = j0 / TH; ty1 = j1 / TH;
    return true;
}

__global__ void __launch_bounds__(256) k3_count(Tables t, BinSet bs, float dil)
{
    const int c = blockIdx.y;
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= t.F) return;
    const Chunk ch = t.chunks[c];
    const ImgInfo &im = t.imgs[ch.b];
    const float4 *r = t.rec + (size_t)(im.rec_off + (long long)ch.s * t.F + f) * REC_F4;
    int tx0, tx1, ty0, ty1;
    if (!swept_tiles(t, r, ch.tmin, ch.tmax, dil, tx0, tx1, ty0, ty1)) return;
    int *cnt = bs.cnt + (size_t)c * t.T;
    for (int ty = ty0; ty <= ty1; ++ty)
        for (int tx = tx0; tx <= tx1; ++tx) atomicAdd(cnt + ty * t.TX + tx, 1);
}

__global__ void __launch_bounds__(256) k3_fill(Tables t, BinSet bs, float dil)
{
    const int c = blockIdx.y;
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= t.F) return;
    const Chunk ch = t.chunks[c];
    const ImgInfo &im = t.imgs[ch.b];
    const float4 *r = t.rec + (size_t)(im.rec_off + (long long)ch.s * t.F + f) * REC_F4;
    int tx0, tx1, ty0, ty1;
    if (!swept_tiles(t, r, ch.tmin, ch.tmax, dil, tx0, tx1, ty0, ty1)) return;
    const size_t base = (size_t)c * t.T;
    bool ovf = false;
    for (int ty = ty0; ty <= ty1; ++ty)
        for (int tx = tx0; tx <= tx1; ++tx) {
            const size_t bi = base + ty * t.TX + tx;
            const long long pos = (long long)bs.off[bi] + atomicAdd(bs.cnt + bi, 1);
            if (pos < bs.cap) bs.entries[pos] = f;
            else ovf = true;
        }
    if (ovf) atomicOr(t.status, BLUR_ST_EOVERFLOW);
}

// Shared-memory variants (images with <= K3_SMEM_TILES tiles): a CTA takes K3_FPB faces of one
// chunk and counts their tiles in a shared histogram, so that the global atomics are one per
// (CTA, touched tile) instead of one per (face, tile) entry; the fill reserves each touched tile's
// range with one global atomic and places the entries with shared cursors.
constexpr int K3_FPB = 1024;
constexpr int K3_SMEM_TILES = 4096;

__global__ void __launch_bounds__(256) k3_count_s(Tables t, BinSet bs, float dil)
{
    extern __shared__ int hist[];   // [T]
    const int c = blockIdx.y, T = t.T;
    for (int i = threadIdx.x; i < T; i += 256) hist[i] = 0;
    __syncthreads();
    const Chunk ch = t.chunks[c];
    const ImgInfo &im = t.imgs[ch.b];
    const int f1 = min(t.F, (int)(blockIdx.x + 1) * K3_FPB);
    for (int f = blockIdx.x * K3_FPB + threadIdx.x; f < f1; f += 256) {
        const float4 *r = t.rec + (size_t)(im.rec_off + (long long)ch.s * t.F + f) * REC_F4;
        int tx0, tx1, ty0, ty1;
        if (!swept_tiles(t, r, ch.tmin, ch.tmax, dil, tx0, tx1, ty0, ty1)) continue;
        for (int ty = ty0; ty <= ty1; ++ty)
            for (int tx = tx0; tx <= tx1; ++tx) atomicAdd(hist + ty * t.TX + tx, 1);
    }
    __syncthreads();
    int *cnt = bs.cnt + (size_t)c * T;
    for (int i = threadIdx.x; i < T; i += 256)
        if (hist[i]) atomicAdd(cnt + i, hist[i]);
}

__global__ void __launch_bounds__(256) k3_fill_s(Tables t, BinSet bs, float dil)
{
    extern __shared__ long long sbase[];   // [T] global start of this CTA's range per tile, then [T] ints
    const int c = blockIdx.y, T = t.T;
    int *hist = reinterpret_cast<int *>(sbase + T);
    for (int i = threadIdx.x; i < T; i += 256) hist[i] = 0;
    __syncthreads();
    const Chunk ch = t.chunks[c];
    const ImgInfo &im = t.imgs[ch.b];
    const int f1 = min(t.F, (int)(blockIdx.x + 1) * K3_FPB);
    for (int f = blockIdx.x * K3_FPB + threadIdx.x; f < f1; f += 256) {
        const float4 *r = t.rec + (size_t)(im.rec_off + (long long)ch.s * t.F + f) * REC_F4;
        int tx0, tx1, ty0, ty1;
        if (!swept_tiles(t, r, ch.tmin, ch.tmax, dil, tx0, tx1, ty0, ty1)) continue;
        for (int ty = ty0; ty <= ty1; ++ty)
            for (int tx = tx0; tx <= tx1; ++tx) atomicAdd(hist + ty * t.TX + tx, 1);
    }
    __syncthreads();
    const size_t base = (size_t)c * T;
    for (int i = threadIdx.x; i < T; i += 256) {
        const int h = hist[i];
        if (h) sbase[i] = bs.off[base + i] + atomicAdd(bs.cnt + base + i, h);
        hist[i] = 0;
    }
    __syncthreads();
    bool ovf = false;
    for (int f = blockIdx.x * K3_FPB + threadIdx.x; f < f1; f += 256) {
        const float4 *r = t.rec + (size_t)(im.rec_off + (long long)ch.s * t.F + f) * REC_F4;
        int tx0, tx1, ty0, ty1;
        if (!swept_tiles(t, r, ch.tmin, ch.tmax, dil, tx0, tx1, ty0, ty1)) continue;
        for (int ty = ty0; ty <= ty1; ++ty)
            for (int tx = tx0; tx <= tx1; ++tx) {
                const int ti = ty * t.TX + tx;
                const long long pos = sbase[ti] + atomicAdd(hist + ti, 1);
                if (pos < bs.cap) bs.entries[pos] = f;
                else ovf = true;
            }
    }
    if (ovf) atomicOr(t.status, BLUR_ST_EOVERFLOW);
}

// ---- exclusive scan of cnt[0..n) into off[0..n], off[n] = total (3 kernels, 1024 per block)
__device__ __forceinline__ int block_excl_scan_1024(int v[4], int *sm)
{
    // 256 threads x 4 items; returns the block total, v[] becomes exclusive prefixes
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int s = v[0] + v[1] + v[2] + v[3];
    int x = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sm[warp] = x;
    __syncthreads();
    if (warp == 0) {
        int w = lane < 8 ? sm[lane] : 0;
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < 8) sm[8 + lane] = w;
    }
    __syncthreads();
    int excl = x - s + (warp > 0 ? sm[8 + warp - 1] : 0);
    int total = sm[8 + 7];
    int run = excl;
#pragma unroll
    for (int i = 0; i < 4; ++i) { int tmp = v[i]; v[i] = run; run += tmp; }
    __syncthreads();
    return total;
}

__global__ void __launch_bounds__(256) k3_scan_blocks(const int *cnt, long long *off, long long *bsum, int n)
{
    __shared__ int sm[16];
    const int base = blockIdx.x * 1024 + threadIdx.x * 4;
    int v[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = base + i < n ? cnt[base + i] : 0;
    int tot = block_excl_scan_1024(v, sm);
#pragma unroll
    for (int i = 0; i < 4; ++i)
        if (base + i < n) off[base + i] = v[i];
    if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

// exclusive scan of the block totals (64-bit), one CTA; off[n] = grand total
__global__ void __launch_bounds__(256) k3_scan_sums(long long *bsum, int nb, long long *off, int n,
                                                    long long *binstat, long long cap)
{
    __shared__ long long sm[16];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    long long carry = 0;
    for (int base0 = 0; base0 < nb; base0 += 256) {
        const int i = base0 + tid;
        const long long v = i < nb ? bsum[i] : 0;
        long long x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) sm[warp] = x;
        __syncthreads();
        long long pre = 0, tot = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w) {
            pre += w < warp ? sm[w] : 0;
            tot += sm[w];
        }
        if (i < nb) bsum[i] = carry + pre + x - v;
        carry += tot;
        __syncthreads();
    }
    if (tid == 0) {
        off[n] = carry;
        binstat[0] = carry;
        binstat[1] = cap;
    }
}

__global__ void __launch_bounds__(256) k3_scan_add(long long *off, const long long *bsum, int n)
{
    const int i = blockIdx.x * 1024 + threadIdx.x;
    const long long add = bsum[blockIdx.x];
#pragma unroll
    for (int q = 0; q < 4; ++q)
        if (i + 256 * q < n) off[i + 256 * q] += add;
}

// ---- per-bin bitonic sort (one warp per bin)
// soft bins: true if every pixel of the bin's tile is covered at every sub-frame of its chunk (K4's
// coverage ballots; out-of-image pixels count as covered) -- no soft term is ever evaluated for it,
// so it need not be sorted.  Warp-uniform.
__device__ __forceinline__ bool bin_fully_covered(const Tables &t, int bi, int lane)
{
    if (!t.covbits) return false;
    const int c = bi / t.T, tile = bi - c * t.T;
    const Chunk ch = t.chunks[c];
    const ImgInfo &im = t.imgs[ch.b];
    const int nw = (ch.k1 - ch.k0) * (NT / 32);
    bool all = true;
    for (int i = lane; i < nw; i += 32) {
        const int k = ch.k0 + i / (NT / 32), w = i % (NT / 32);
        all &= t.covbits[cov_word(t, im, k, tile) + w] == 0xFFFFFFFFu;
    }
    return __all_sync(0xffffffffu, all);
}

__global__ void __launch_bounds__(256) k3_sort(Tables t, BinSet bs, int nbins)
{
    __shared__ int sm[8][SORTCAP];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int *s = sm[warp];
    for (int bi = blockIdx.x * 8 + warp; bi < nbins; bi += gridDim.x * 8) {
        const long long o = bs.off[bi];
        const int n = (int)(bs.off[bi + 1] - o);
        if (n <= 1 || n > SORTCAP || o + n > bs.cap) continue;
        if (bin_fully_covered(t, bi, lane)) continue;
        int n2 = 32;
        while (n2 < n) n2 <<= 1;
        for (int i = lane; i < n2; i += 32) s[i] = i < n ? bs.entries[o + i] : 0x7fffffff;
        __syncwarp();
        for (int k = 2; k <= n2; k <<= 1)
            for (int j = k >> 1; j > 0; j >>= 1) {
                for (int i = lane; i < n2; i += 32) {
                    const int ixj = i ^ j;
                    if (ixj > i) {
                        const int a = s[i], b = s[ixj];
                        const bool up = (i & k) == 0;
                        if ((a > b) == up) { s[i] = b; s[ixj] = a; }
                    }
                }
                __syncwarp();
            }
        // self-check: a sorted bin holds distinct ids in [0, F)
        bool bad = false;
        for (int i = lane; i < n; i += 32) {
            bs.entries[o + i] = s[i];
            bad |= s[i] < 0 || s[i] >= t.F || (i > 0 && s[i - 1] >= s[i]);
        }
        if (__any_sync(0xffffffffu, bad) && lane == 0) {
            atomicOr(t.status, BLUR_ST_EINTERNAL);
#ifdef BR_DEBUG
            printf("bad sorted bin %d o=%d n=%d: %d %d %d %d ... last %d\n", bi, o, n, s[0], s[1], s[2], s[3], s[n - 1]);
#endif
        }
        __syncwarp();
    }
}

// ---- CTA-per-bin bitonic sort of the bins longer than SORTCAP (soft bins, up to bs.sortcap <= SORTCAP_BIG):
// the bin in dynamic shared memory (64 KB at 16384 entries).  Longer soft bins take the raster kernels' exact
// fallback, a scan of every face of the segment per (sub-frame, tile): on C5 (1024^2, 81,920 faces, rcut = 21
// px) the silhouette tiles' soft bins exceed 4,096 entries, and that scan was most of K8/K9's time.
constexpr int SORTCAP_BIG = 16384;
__global__ void __launch_bounds__(512) k3_sort_big(Tables t, BinSet bs, int nbins)
{
    extern __shared__ int s[];   // [SORTCAP_BIG]
    __shared__ int bad;
    for (int bi = blockIdx.x; bi < nbins; bi += gridDim.x) {
        const long long o = bs.off[bi];
        const int n = (int)(bs.off[bi + 1] - o);
        if (n <= SORTCAP || n > bs.sortcap || o + n > bs.cap) continue;   // block-uniform
        {
            __shared__ int cov;
            if (threadIdx.x < 32) {
                const bool fc = bin_fully_covered(t, bi, threadIdx.x);
                if (threadIdx.x == 0) cov = fc;
            }
            __syncthreads();
            const bool skip = cov;
            __syncthreads();
            if (skip) continue;
        }
        int n2 = 2 * SORTCAP;
        while (n2 < n) n2 <<= 1;
        if (threadIdx.x == 0) bad = 0;
        for (int i = threadIdx.x; i < n2; i += blockDim.x) s[i] = i < n ? bs.entries[o + i] : 0x7fffffff;
        __syncthreads();
        for (int k = 2; k <= n2; k <<= 1)
            for (int j = k >> 1; j > 0; j >>= 1) {
                for (int i = threadIdx.x; i < n2; i += blockDim.x) {
                    const int ixj = i ^ j;
                    if (ixj > i) {
                        const int a = s[i], b = s[ixj];
                        const bool up = (i & k) == 0;
                        if ((a > b) == up) { s[i] = b; s[ixj] = a; }
                    }
                }
                __syncthreads();
            }
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            bs.entries[o + i] = s[i];
            if (s[i] < 0 || s[i] >= t.F || (i > 0 && s[i - 1] >= s[i])) bad = 1;
        }
        __syncthreads();
        if (threadIdx.x == 0 && bad) atomicOr(t.status, BLUR_ST_EINTERNAL);
        __syncthreads();
    }
}

cudaError_t launch_binning(const Tables &t, const BinSet &bs, float dil, cudaStream_t st)
{
    const int nbins = t.NC * t.T;
    if (nbins == 0) return cudaSuccess;
    cudaError_t e = cudaMemsetAsync(bs.cnt, 0, sizeof(int) * (size_t)nbins, st);
    if (e != cudaSuccess) return e;
    const bool shm = t.T <= K3_SMEM_TILES;
    if (t.F > 0) {
        if (shm) {
            dim3 grid((t.F + K3_FPB - 1) / K3_FPB, t.NC);
            k3_count_s<<<grid, 256, sizeof(int) * t.T, st>>>(t, bs, dil);
        } else {
            dim3 grid((t.F + 255) / 256, t.NC);
            k3_count<<<grid, 256, 0, st>>>(t, bs, dil);
        }
    }
    const int nb = (nbins + 1023) / 1024;
    k3_scan_blocks<<<nb, 256, 0, st>>>(bs.cnt, bs.off, bs.bsum, nbins);
    k3_scan_sums<<<1, 256, 0, st>>>(bs.bsum, nb, bs.off, nbins, bs.binstat, bs.cap);
    k3_scan_add<<<nb, 256, 0, st>>>(bs.off, bs.bsum, nbins);
    e = cudaMemsetAsync(bs.cnt, 0, sizeof(int) * (size_t)nbins, st);
    if (e != cudaSuccess) return e;
    if (t.F > 0) {
        if (shm) {
            const size_t smem = (sizeof(long long) + sizeof(int)) * t.T;
            e = cudaFuncSetAttribute(k3_fill_s, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess) return e;
            dim3 grid((t.F + K3_FPB - 1) / K3_FPB, t.NC);
            k3_fill_s<<<grid, 256, smem, st>>>(t, bs, dil);
        } else {
            dim3 grid((t.F + 255) / 256, t.NC);
            k3_fill<<<grid, 256, 0, st>>>(t, bs, dil);
        }
        int sb = (nbins + 7) / 8;
        if (sb > 148 * 16) sb = 148 * 16;
        if (bs.sortcap > 0) k3_sort<<<sb, 256, 0, st>>>(t, bs, nbins);
        if (bs.sortcap > SORTCAP) {
            const int smem = (int)sizeof(int) * SORTCAP_BIG;
            e = cudaFuncSetAttribute(k3_sort_big, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            if (e != cudaSuccess) return e;
            k3_sort_big<<<std::min(nbins, 148 * 2), 512, smem, st>>>(t, bs, nbins);
        }
    }
    return cudaGetLastError();
}

}  // namespace br
