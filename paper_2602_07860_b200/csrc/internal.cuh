// internal.cuh -- device-side layouts shared by the kernels of libblurrast (not part of the ABI).
// See include/blurrast.h for the public contract and DESIGN.md for the data layout in HBM.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace br {

// Tile geometry of the raster kernels: a CTA owns a TW x TH pixel tile; each warp owns an
// 8 x 4 footprint (8 warps).  One pixel per thread.
constexpr int TW = 16;
constexpr int TH = 16;
constexpr int NT = 256;          // threads per raster CTA
constexpr int CAP = 512;         // per-(tile, sub-frame) face records staged per batch (smem)
constexpr int SORTCAP = 1024;    // bins longer than this take the exact fallback path
constexpr float EPS_D = 1e-12f;  // Q8: |det F| <= 1e-12 NDC^2 -> face skipped for that sub-frame
constexpr float BBOX_PAD = 1e-5f;  // NDC padding of conservative bounding boxes (>> fp32 error)
constexpr int VIS_MAXN = 256;    // bins of at most this many faces get K4's visibility cache (BLUR_CACHE_VISIBILITY)

// Per (face, segment) coefficient record: the paper's Eq.8 coefficients (A1, A2, A3, a1..a3),
// computed once per segment, in edge-vector form about a per-edge origin (DESIGN.md
// "edge-vector form"), plus the depth keyframes and conservative keyframe bounding boxes.
// 44 floats = 11 x float4 = 176 B.
//   [8i+0..8i+7]  numerator of w_i (edge opposite corner i): ox, oy, a0, a1, b0, b1, dax, day
//                 N_i(tau; p) = (a0 + a1 tau)(u - ax(tau)) + (b0 + b1 tau)(v - ay(tau)),
//                 a(tau) = (ox + tau dax, oy + tau day) the edge's canonical start vertex at tau (Eq.5-6):
//                 the Eq.8 polynomial A1 tau^2 + A2(p) tau + A3(p) in factored form, with
//                 A1_i = -(a1 dax + b1 day), A2_i(p) = a1 (u-ox) + b1 (v-oy) - (a0 dax + b0 day),
//                 A3_i(p) = a0 (u-ox) + b0 (v-oy).  Evaluated about the moving vertex, the pixel offsets
//                 stay of the size of the triangle however far it travels in the segment (the expanded
//                 form cancels terms of the size of the travel: 20x the fp32 error of a limb sliver on C4)
//   [24..26]      d1, d2, d3: det F(tau) = d3 + tau (d2 + tau d1)  (a1, a2, a3 of Eq.8)
//   [27]          face id (int bits), -1 = skipped face
//   [28..31]      bbox at keyframe s (xmin, xmax, ymin, ymax), [32..35] at keyframe s+1 (padded)
//   [36..38]      view depth at keyframe s, [40..42] at keyframe s+1 ([39], [43] unused)
constexpr int REC_F4 = 11;
constexpr int REC_FLOATS = 44;

struct ImgInfo {
    int N, S;            // sub-frames, segments
    int k0, k1;          // sub-frame range [k0, k1)
    int sched_off;       // offset of this image's schedule in the sched arrays
    int key_off;         // offset (float4 units) of keyframes [S+1][V]; also float2 offset of dkey
    long long rec_off;   // offset (records) of coefficient records [S][F]
    int chunk_begin, chunk_end;
    int pose_off;        // offset (in PoseRec) of keyframe poses [S+1]
    int cov_off;         // soft path: offset (sub-frames) of this image's coverage words
    double Rc[9];        // camera rotation rows (right, up', forward)
    double eye[3];
    double tan_half;     // tan(half_fov)
    double z_near;
};

struct PoseRec {         // P = R (P0 - c) + c + T at keyframe time t = s/S
    double R[9];
    double c[3];
    double T[3];
};

struct Chunk {           // consecutive sub-frames of one image inside one segment
    int b, s, k0, k1;    // sub-frames k0..k1-1 (image-local indices)
    float tmin, tmax;    // tau of the first / last sub-frame
};

struct BinSet {          // one set of (chunk, tile) bins (K3): counters, offsets, sorted entries
    int *cnt;            // [NC * T]
    long long *off;      // [NC * T + 1] bin offsets (64-bit: large batches exceed 2^31 entries)
    long long *bsum;     // scan block sums
    int *entries;        // bin entries (face ids)
    long long cap;       // entries capacity
    long long *binstat;  // [0] entries the last binning needed, [1] capacity
    int sortcap;         // bins longer than this are not sorted (raster kernels take the exact fallback)
};

struct Tables {          // device pointers into the workspace
    int *status;
    long long *binstat;  // [0] bin entries the last binning needed, [1] entry capacity
    const ImgInfo *imgs;
    const Chunk *chunks;
    const int *sched_s;
    const float *sched_tau;
    const PoseRec *poses;
    float4 *key;         // keyframes (x_ndc, y_ndc, z_view, valid)
    float4 *rec;         // coefficient records
    float4 *fcol;        // per face: 3 x float4 = c0.rgb c1.rgb c2.rgb vid0 vid1 vid2 (int bits)
    int *cnt;            // [NC * T]
    long long *off;      // [NC * T + 1] bin offsets (64-bit: large batches exceed 2^31 entries)
    long long *bsum;     // scan block sums
    int *entries;        // bin entries (face ids)
    long long cap;       // entries capacity
    float2 *dkey;        // screen-space keyframe gradients, indexed like key
    int NC, T, TX, TY;
    int B, V, F, H, W;
    int solver;          // 0 fast (Eq.8 coefficients), 1 naive per-frame setup, 2 naive per-pixel solve
    int legacy;          // 1: the fast solver also takes k_raster.cu's footprint-mask kernels (A/B only)
    int splits;          // CTAs sharing one (image, tile) by sub-frame chunks (small launches)
    int ssplits;         // the same for the soft kernels K8/K9 (>= splits: their silhouette tiles
                         // are heavy, so splitting them shortens the launch's tail)
    float4 *part;        // splits > 1: per-split partial images [splits][B*H*W]
    // soft background coverage (NEXT-1; delta > 0)
    float delta;         // Eq.10 bandwidth (NDC^2)
    float rcut;          // NDC radius beyond which a face's term is dropped: sqrt(soft_cut * delta)
    float rcut_f;        // the forward's radius sqrt(min(soft_cut, 18) delta): farther factors are 1.0f
    int soft_exact;      // 1: Eq.12 (closest point on F(tau)) instead of Eq.13 (on F(X))
    uint32_t *covbits;   // [sum_b N_b][T][NWARP] coverage ballots per (sub-frame, tile, warp) or null
    uint16_t *vis;       // [sum_b N_b][T][TW*TH] winning bin slot per (sub-frame, pixel), 0xFFFF none;
                         // written by K4, read by K6 instead of recomputing visibility (or null)
    double *orient;      // mesh orientation: sum over faces of det(P0[v0], P0[v1], P0[v2]) (6 x signed volume;
                         // > 0: outward counter-clockwise faces), written by the setup (k_orient)
    int vis_gathered;    // 1: k6v_raster_bwd (k_gather.cu) has taken the cached chunks; k6_raster_bwd_fx skips them
    int *vg_count;       // k6v_raster_bwd: number of (image, tile)s with chunks left to k6_raster_bwd_fx,
    int *vg_list;        // ... and their b * T + tile ([B * T])
    float *spart;        // [splits][B*H*W] soft alpha partial sums (K8)
    float *spz;          // [sum_b N_b][T][TW*TH] soft products per (sub-frame, pixel) left by K8 for K9
                         // (prod of the non-zero factors 1 - A; negative: one zero factor, NaN: two or
                         // more; written where K8 needs the pixel) or null
    BinSet sb;           // soft bins (chunk boxes dilated by rcut)
};

struct __align__(16) TauRec {    // per (face, sub-frame, tile) staged record, 64 B
    float a[3], b[3], g[3];      // sign-normalised edge functions: e_i = a_i ul + b_i vl + g_i
    float az, bz, cz;            // view depth plane in tile-local coordinates
    float invD;                  // 1 / |det F(tau)|
    int fid;
    int pad0, pad1;
};

// NDC interval -> inclusive pixel-centre index range (Q9: centre of pixel i at -1 + (2i+1)/W).
// Explicit-rounding arithmetic so that every kernel (K3 binning, raster staging, fallback scan)
// derives bit-identical ranges from identical inputs (no compiler-chosen FMA contraction).
__device__ __forceinline__ void ndc_to_index(float lo, float hi, int n, bool flip, float &a, float &b)
{
    const float fn = (float)n;
    if (!flip) {   // x: i >= ((lo + 1) n - 1) / 2
        a = ceilf(__fmul_rn(__fsub_rn(__fmul_rn(__fadd_rn(lo, 1.f), fn), 1.f), 0.5f));
        b = floorf(__fmul_rn(__fsub_rn(__fmul_rn(__fadd_rn(hi, 1.f), fn), 1.f), 0.5f));
    } else {       // y (row 0 at the top): j >= ((1 - hi) n - 1) / 2
        a = ceilf(__fmul_rn(__fsub_rn(__fmul_rn(__fsub_rn(1.f, hi), fn), 1.f), 0.5f));
        b = floorf(__fmul_rn(__fsub_rn(__fmul_rn(__fsub_rn(1.f, lo), fn), 1.f), 0.5f));
    }
}

// soft path: first of the NWARP coverage words of (image, sub-frame k, tile)
__device__ __forceinline__ size_t cov_word(const Tables &t, const ImgInfo &im, int k, int tile)
{
    return ((size_t)(im.cov_off + k) * t.T + tile) * (NT / 32);
}

// Edge i of a K2 record at tau (qa = record float4 2i, qb = 2i+1): d/du and d/dv of N_i and its value at
// (uc, vc), N_i = al (uc - ax(tau)) + be (vc - ay(tau)).  Every kernel evaluates records through this one
// helper, so the two faces of an edge (same canonical data, sign flipped) get exact negations: watertight.
__device__ __forceinline__ void rec_edge_at(const float4 qa, const float4 qb, float tau, float uc, float vc, float &al,
                                            float &be, float &gp)
{
    al = __fmaf_rn(tau, qa.w, qa.z);
    be = __fmaf_rn(tau, qb.y, qb.x);
    const float ax = __fmaf_rn(tau, qb.z, qa.x), ay = __fmaf_rn(tau, qb.w, qa.y);
    gp = __fmaf_rn(al, __fsub_rn(uc, ax), __fmul_rn(be, __fsub_rn(vc, ay)));
}

// Checked build (-DBR_CHECKED, tools/checked_build.sh): shared-memory index invariants of the raster kernels
// are tested at run time and a violation raises BLUR_ST_EINTERNAL (surfaced by blur_read_status /
// BLURRAST_CHECK=1) -- the memory-safety evidence this pool allows in place of compute-sanitizer.
#ifdef BR_CHECKED
#define BR_CHECK(cond, status_ptr) do { if (!(cond)) atomicOr((status_ptr), 8); } while (0)
#else
#define BR_CHECK(cond, status_ptr) ((void)0)
#endif

// conservative keyframe box lerped to tau (monotone in tau for fixed endpoints)
__device__ __forceinline__ float box_lerp(float tau, float a, float b) { return __fmaf_rn(tau, __fsub_rn(b, a), a); }

}  // namespace br

// launchers (defined in the .cu files)
#include <string>
namespace br {
void set_last_error(const std::string &msg);   // thread-local message of blur_last_error() (abi.cu)
void clear_last_error();
cudaError_t launch_setup(const Tables &t, const float *verts, const int *faces, const float *colors,
                         int maxS, cudaStream_t st);
cudaError_t launch_binning(const Tables &t, const BinSet &bs, float dil, cudaStream_t st);
cudaError_t launch_soft_fwd(const Tables &t, float *out, unsigned long long *census, cudaStream_t st);
cudaError_t launch_soft_bwd(const Tables &t, const float *grad_rgba, cudaStream_t st);
cudaError_t launch_raster_fwd(const Tables &t, float *out, int *ids, int ids_k,
                              unsigned long long *census, cudaStream_t st);
cudaError_t launch_raster_bwd(const Tables &t, const float *grad_rgba, float *grad_colors,
                              cudaStream_t st);
// round-1 footprint-mask raster kernels (k_raster.cu): the naive solvers of the NEXT-2 ablation, and the
// fast solver when Tables::legacy is set (A/B)
cudaError_t launch_raster_fwd_legacy(const Tables &t, float *out, int *ids, int ids_k,
                                     unsigned long long *census, cudaStream_t st);
cudaError_t launch_raster_bwd_legacy(const Tables &t, const float *grad_rgba, float *grad_colors,
                                     cudaStream_t st);
// K4 in the pixel-major evaluation order (k_pixmajor.cu; BLURRAST_FWD=pixmajor, A/B only)
bool pixmajor_fwd_on();
cudaError_t launch_raster_fwd_pixmajor(const Tables &t, float *out, int *ids, int ids_k, cudaStream_t st);
cudaError_t launch_vis_gather(const Tables &t, const float *grad_rgba, float *grad_colors, cudaStream_t st);
cudaError_t launch_vertex_chain(const Tables &t, float *grad_verts, cudaStream_t st);
cudaError_t launch_split_reduce(const Tables &t, float *out, cudaStream_t st);
cudaError_t launch_l2(const float *out, const float *tgt, long long n, long long n_norm, float *loss,
                      float *grad, cudaStream_t st);
cudaError_t launch_ffma_probe(int ctas, int iters, float *sink, cudaStream_t st);
// p / ng for the (face, sub-frame) pair loops without an integer division: p < 2^13 and ng <= 16,
// so (p + 0.5) / ng in fp32 (relative error < 1e-6) is never within rounding of an integer
__device__ __forceinline__ int div_small(int p, float inv_ng) { return __float2int_rz(((float)p + 0.5f) * inv_ng); }

// floor(cap / n) for 1 <= n <= cap <= 4096 without an integer division: cap / n is either an integer
// (exact in fp32) or at least 1 / n below the next one, far more than __fdividef's 2-ulp error
__device__ __forceinline__ int group_div(int cap, int n) { return (int)__fdividef((float)cap, (float)n); }

}  // namespace br
