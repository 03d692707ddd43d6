// abi.cu -- the C ABI of libblurrast (include/blurrast.h): argument validation, the host-side
// schedule/pose/chunk plan (L0), workspace carving and the launch sequence K1..K7.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>   // header-only NVTX3: ranges cost a branch unless a tool (nsys, ncu --nvtx) attaches

#include "internal.cuh"
#include "../../include/blurrast.h"

#ifndef BR_HARD_SPLITS
#define BR_HARD_SPLITS 2   // hard raster: at least 2 CTAs per (image, tile) when it has 2+ chunks (C4 -1%)
#endif
#ifndef BR_K8_CUT
#define BR_K8_CUT 18.f     // K8's cut in units of delta (see rcut_f)
#endif
#ifndef BR_SOFT_SPLITS
#define BR_SOFT_SPLITS 8   // soft kernels: up to 8 CTAs per (image, tile), each taking every 8th chunk
#endif

using namespace br;

namespace {

thread_local std::string g_err;

// NVTX range over a scope: the ABI calls and their phases (setup, binning, raster, soft, vertex chain) show up
// by name on a profiler timeline (`ncu --nvtx --nvtx-include "blur_render_fwd/"`)
struct Nvtx {
    explicit Nvtx(const char *name) { nvtxRangePushA(name); }
    ~Nvtx() { nvtxRangePop(); }
    Nvtx(const Nvtx &) = delete;
    Nvtx &operator=(const Nvtx &) = delete;
};

int fail(int code, const std::string &msg)
{
    g_err = msg;
    return code;
}

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

// Q1 schedule (same reading as DESIGN.md; integer arithmetic for GLOBAL_INCLUSIVE)
bool schedule(int N, int S, int rule, std::vector<int> &s_out, std::vector<float> &tau_out)
{
    s_out.resize(N);
    tau_out.resize(N);
    if (rule == BLUR_SCHED_PAPER_SEGMENTED) {
        if (N % S) return false;
        const int K = N / S;
        for (int k = 0; k < N; ++k) {
            s_out[k] = k / K;
            tau_out[k] = K == 1 ? 0.5f : (float)((double)(k % K) / (double)(K - 1));
        }
        return true;
    }
    if (rule != BLUR_SCHED_GLOBAL_INCLUSIVE) return false;
    if (N == 1) {
        int s = S / 2;
        if (s > S - 1) s = S - 1;
        s_out[0] = s;
        tau_out[0] = (float)(0.5 * S - s);
        return true;
    }
    for (int k = 0; k < N; ++k) {
        const long long num = (long long)k * S;
        long long s = num / (N - 1);
        if (s > S - 1) s = S - 1;
        s_out[k] = (int)s;
        tau_out[k] = (float)((double)(num - s * (N - 1)) / (double)(N - 1));
    }
    return true;
}

void rodrigues(const double ax_in[3], double th, double R[9])
{
    double a[3] = {ax_in[0], ax_in[1], ax_in[2]};
    const double n = std::sqrt(a[0] * a[0] + a[1] * a[1] + a[2] * a[2]);
    for (double &x : a) x /= n;
    const double K[9] = {0, -a[2], a[1], a[2], 0, -a[0], -a[1], a[0], 0};
    const double sn = std::sin(th), cs = 1.0 - std::cos(th);
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double k2 = 0;
            for (int l = 0; l < 3; ++l) k2 += K[i * 3 + l] * K[l * 3 + j];
            R[i * 3 + j] = (i == j ? 1.0 : 0.0) + sn * K[i * 3 + j] + cs * k2;
        }
}

struct Plan {
    int B = 0, V = 0, F = 0, H = 0, W = 0, TX = 0, TY = 0, T = 0, NC = 0, maxS = 1, splits = 1, ssplits = 1;
    std::vector<ImgInfo> imgs;
    std::vector<Chunk> chunks;
    std::vector<int> sched_s;
    std::vector<float> sched_tau;
    std::vector<PoseRec> poses;
    long long n_key = 0, n_rec = 0, cap = 0;
    size_t nbins = 0;
    size_t o_status = 0, o_imgs = 0, o_chunks = 0, o_ss = 0, o_st = 0, o_poses = 0, o_tables_end = 0;
    size_t o_key = 0, o_rec = 0, o_fcol = 0, o_cnt = 0, o_off = 0, o_bsum = 0, o_ent = 0, o_dkey = 0, o_part = 0;
    // soft background coverage (NEXT-1)
    bool soft = false;
    float delta = 0.f, rcut = 0.f, rcut_f = 0.f;
    int soft_exact = 0;
    long long scap = 0, n_sub = 0;
    size_t o_cov = 0, o_spart = 0, o_scnt = 0, o_soff = 0, o_sbsum = 0, o_sent = 0;
    bool vis = false;      // BLUR_CACHE_VISIBILITY: K4 leaves the winning bin slot per (pixel, sub-frame)
    size_t o_vis = 0;
    size_t o_vgl = 0;      // visibility gather: count + list of the (image, tile)s it left to k6_raster_bwd_fx
    size_t o_spz = 0;      // soft products K8 -> K9 (BLUR_CACHE_VISIBILITY with delta > 0)
    bool spz_on = false;
    size_t total = 0;
};

bool legacy_env();

#ifndef BR_CHUNK2_TILES
#define BR_CHUNK2_TILES 3.5   // 2-sub-frame chunks up to 3.5 tiles of motion per sub-frame (C3 2.80 -> 2.56 ms/step
#endif                        // with the lean K4; 1.5 was fitted to round 1's kernel; C2, C4, C5 unchanged)
int auto_chunk(const blur_motion &m, const blur_camera &c, int H, int W)
{
    const double dx = c.eye[0] - c.target[0], dy = c.eye[1] - c.target[1], dz = c.eye[2] - c.target[2];
    const double dist = std::sqrt(dx * dx + dy * dy + dz * dz);
    const double ndc_per_world = 1.0 / (dist * std::tan((double)c.half_fov));
    const double px_per_ndc = 0.5 * (H > W ? H : W);
    const int N = m.n_subframes;
    if (N <= 1) return 16;
    double world = 0.0;
    if (m.kind == BLUR_TRANSLATE)
        world = std::sqrt((double)m.vec[0] * m.vec[0] + (double)m.vec[1] * m.vec[1] + (double)m.vec[2] * m.vec[2]);
    else if (m.kind == BLUR_ROTATE)
        world = std::fabs((double)m.angle);   // unit-size object
    else if (m.kind == BLUR_PARABOLIC)
        world = std::fabs((double)m.angle) + 2.0;
    const double disp = world * ndc_per_world * px_per_ndc / (N - 1);
    if (disp <= 1e-6) return 16;
    // chunk ~ one tile of motion; at least 2 sub-frames unless the motion exceeds BR_CHUNK2_TILES tiles per
    // sub-frame (then per-sub-frame bins); at most 8 (rule fitted on C2-C5: tools/chunk_sweep.sh)
    int g = (int)std::floor(TW / disp);
    if (disp <= BR_CHUNK2_TILES * TW && g < 2) g = 2;
    if (g < 1) g = 1;
    if (g > 8) g = 8;
    return g;
}

int make_plan(int V, int F, int B, int H, int W, const blur_motion *m, const blur_camera *cams,
              const int32_t *sub_range, const blur_config *cfg, Plan &P)
{
    if (V < 0 || F < 0 || B < 0) return fail(BLUR_EINVAL, "V, F, B must be >= 0");
    if (F > 0 && V == 0) return fail(BLUR_EINVAL, "faces given but V == 0");
    if (F > 4000000) return fail(BLUR_EINVAL, "F > 4,000,000 (the raster z-buffer key holds 22 bits of face index)");
    if (H < 1 || W < 1 || H > 32768 || W > 32768) return fail(BLUR_EINVAL, "H, W must be in [1, 32768]");
    if (B > 0 && !m) return fail(BLUR_EINVAL, "motions is NULL");
    P.B = B; P.V = V; P.F = F; P.H = H; P.W = W;
    P.TX = (W + TW - 1) / TW;
    P.TY = (H + TH - 1) / TH;
    P.T = P.TX * P.TY;
    P.imgs.resize(B);
    int key_off = 0;
    long long rec_off = 0;
    for (int b = 0; b < B; ++b) {
        const blur_motion &mo = m[b];
        const int N = mo.n_subframes;
        int S = mo.n_segments;
        if (S == 0) {   // automatic (Q24): 1 for translation / static, 12 per full turn for rotation
            S = 1;
            if (mo.kind == BLUR_ROTATE || mo.kind == BLUR_PARABOLIC)
                S = std::max(1, (int)std::ceil(12.0 * (std::fabs((double)mo.angle) / (2.0 * M_PI)) - 1e-6));
        }
        if (mo.kind < 0 || mo.kind > 3) return fail(BLUR_EINVAL, "motion kind must be 0, 1, 2 or 3");
        if (N < 1) return fail(BLUR_EINVAL, "n_subframes must be >= 1");
        if (S < 1) return fail(BLUR_EINVAL, "n_segments must be >= 1");
        if (mo.sched_rule == BLUR_SCHED_PAPER_SEGMENTED && N % S)
            return fail(BLUR_EINVAL, "PAPER_SEGMENTED needs n_segments | n_subframes");
        if (mo.sched_rule != 0 && mo.sched_rule != 1) return fail(BLUR_EINVAL, "bad sched_rule");
        if (mo.kind == BLUR_ROTATE || mo.kind == BLUR_PARABOLIC) {
            const double n = std::sqrt((double)mo.vec[0] * mo.vec[0] + (double)mo.vec[1] * mo.vec[1] +
                                       (double)mo.vec[2] * mo.vec[2]);
            if (!(n > 0)) return fail(BLUR_EINVAL, "rotation axis is zero");
        }
        if (!std::isfinite(mo.angle) || !std::isfinite(mo.vec[0]) || !std::isfinite(mo.vec[1]) ||
            !std::isfinite(mo.vec[2]))
            return fail(BLUR_EINVAL, "non-finite motion parameter");
        if (S > P.maxS) P.maxS = S;
        ImgInfo &im = P.imgs[b];
        std::memset(&im, 0, sizeof(im));
        im.N = N;
        im.S = S;
        im.k0 = sub_range ? sub_range[2 * b] : 0;
        im.k1 = sub_range ? sub_range[2 * b + 1] : N;
        if (im.k0 < 0 || im.k1 > N || im.k0 > im.k1) return fail(BLUR_EINVAL, "sub_range out of [0, N]");
        im.sched_off = (int)P.sched_s.size();
        std::vector<int> ss;
        std::vector<float> tt;
        if (!schedule(N, S, mo.sched_rule, ss, tt)) return fail(BLUR_EINVAL, "invalid schedule");
        P.sched_s.insert(P.sched_s.end(), ss.begin(), ss.end());
        P.sched_tau.insert(P.sched_tau.end(), tt.begin(), tt.end());
        im.key_off = key_off;
        key_off += (S + 1) * V;
        im.cov_off = (int)P.n_sub;
        P.n_sub += N;
        im.rec_off = rec_off;
        rec_off += (long long)S * F;
        // camera
        const blur_camera &c = cams[b];
        if (!(c.half_fov > 0.f && c.half_fov < 1.5707963f)) return fail(BLUR_EINVAL, "half_fov not in (0, pi/2)");
        if (!(c.z_near > 0.f)) return fail(BLUR_EINVAL, "z_near must be > 0");
        double f[3] = {(double)c.target[0] - c.eye[0], (double)c.target[1] - c.eye[1], (double)c.target[2] - c.eye[2]};
        double fn = std::sqrt(f[0] * f[0] + f[1] * f[1] + f[2] * f[2]);
        if (!(fn > 0)) return fail(BLUR_EINVAL, "eye == target");
        for (double &x : f) x /= fn;
        double r[3] = {f[1] * c.up[2] - f[2] * c.up[1], f[2] * c.up[0] - f[0] * c.up[2], f[0] * c.up[1] - f[1] * c.up[0]};
        double rn = std::sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
        double upn = std::sqrt((double)c.up[0] * c.up[0] + (double)c.up[1] * c.up[1] + (double)c.up[2] * c.up[2]);
        if (!(rn > 1e-9 * upn) || !(upn > 0)) return fail(BLUR_EINVAL, "up parallel to the view direction");
        for (double &x : r) x /= rn;
        const double u[3] = {r[1] * f[2] - r[2] * f[1], r[2] * f[0] - r[0] * f[2], r[0] * f[1] - r[1] * f[0]};
        for (int i = 0; i < 3; ++i) { im.Rc[i] = r[i]; im.Rc[3 + i] = u[i]; im.Rc[6 + i] = f[i]; im.eye[i] = c.eye[i]; }
        im.tan_half = std::tan((double)c.half_fov);
        im.z_near = c.z_near;
        // keyframe poses t = s/S
        im.pose_off = (int)P.poses.size();
        for (int s = 0; s <= S; ++s) {
            PoseRec pr;
            std::memset(&pr, 0, sizeof(pr));
            const double t = (double)s / (double)S;
            for (int i = 0; i < 3; ++i) pr.R[4 * i] = 1.0;
            if (mo.kind == BLUR_TRANSLATE) {
                for (int i = 0; i < 3; ++i) pr.T[i] = (t - 0.5) * (double)mo.vec[i];
            } else if (mo.kind == BLUR_ROTATE || mo.kind == BLUR_PARABOLIC) {
                const double ax[3] = {mo.vec[0], mo.vec[1], mo.vec[2]};
                rodrigues(ax, (double)mo.angle * t, pr.R);
                for (int i = 0; i < 3; ++i) pr.c[i] = mo.pivot[i];
                if (mo.kind == BLUR_PARABOLIC) {    // A36: T(t) = (s, -4 s^2 + 0.5, s), s = 0.5 - t
                    const double sp = 0.5 - t;
                    pr.T[0] = sp;
                    pr.T[1] = -4.0 * sp * sp + 0.5;
                    pr.T[2] = sp;
                }
            }
            P.poses.push_back(pr);
        }
        // chunks: runs of consecutive sub-frames in one segment, at most G long
        const int G = (cfg && cfg->max_chunk > 0) ? cfg->max_chunk : auto_chunk(mo, c, H, W);
        im.chunk_begin = (int)P.chunks.size();
        int k = im.k0;
        while (k < im.k1) {
            const int s = ss[k];
            int e = k + 1;
            while (e < im.k1 && ss[e] == s && e - k < G) ++e;
            Chunk ch;
            ch.b = b; ch.s = s; ch.k0 = k; ch.k1 = e;
            ch.tmin = tt[k];
            ch.tmax = tt[e - 1];
            P.chunks.push_back(ch);
            k = e;
        }
        im.chunk_end = (int)P.chunks.size();
    }
    P.NC = (int)P.chunks.size();
    if (P.NC > 65535)   // K3 launches one grid row per chunk (gridDim.y <= 65535)
        return fail(BLUR_EINVAL, "more than 65535 sub-frame chunks in the batch (reduce B x N or raise max_chunk)");
    // each tile's sub-frame chunks are split over BR_HARD_SPLITS CTAs (more for small launches, few
    // tiles x images, so that the grid fills the 148 SMs); partial images are reduced in a fixed
    // order (deterministic).  The soft kernels split further (their silhouette tiles are heavy).
    {
        int maxc = 1;
        for (const ImgInfo &im : P.imgs) maxc = std::max(maxc, im.chunk_end - im.chunk_begin);
        const long long ctas = (long long)P.T * B, target = 148LL * 8;
        P.splits = std::min(maxc, BR_HARD_SPLITS);
        if (ctas > 0 && ctas < target) {
            long long sp = (target + ctas - 1) / ctas;
            if (sp > maxc) sp = maxc;
            if (sp > 32) sp = 32;
            P.splits = (int)std::max(1LL, sp);
        }
        P.ssplits = std::max(P.splits, std::min(maxc, BR_SOFT_SPLITS));
    }
    P.n_key = key_off;
    P.n_rec = rec_off;
    // soft background coverage (NEXT-1): bandwidth, cut-off radius, capacity of the grown bins
    if (cfg && cfg->delta != 0.f) {
        if (!(cfg->delta > 0.f) || !std::isfinite(cfg->delta)) return fail(BLUR_EINVAL, "delta must be >= 0 and finite");
        if (cfg->solver != 0) return fail(BLUR_EINVAL, "soft coverage (delta > 0) needs solver 0");
        const float kc = cfg->soft_cut > 0.f ? cfg->soft_cut : 18.f;
        if (!std::isfinite(kc)) return fail(BLUR_EINVAL, "soft_cut must be finite");
        P.soft = true;
        P.delta = cfg->delta;
        P.rcut = (float)std::sqrt((double)kc * (double)cfg->delta) + 2.0f * BBOX_PAD;
        // K8's own radius: a face at d >= 18 delta from a pixel has A = exp(-d / delta) < 2^-25, so
        // its factor 1 - A rounds to exactly 1.0f and dropping it leaves the products bit-identical
        P.rcut_f = (float)std::sqrt((double)std::min(kc, BR_K8_CUT) * (double)cfg->delta) + 2.0f * BBOX_PAD;
        P.soft_exact = cfg->soft_exact ? 1 : 0;
        const double sf = cfg->soft_bin_factor > 0.f ? cfg->soft_bin_factor : 12.0;
        double sc = sf * (double)P.NC * (double)F + 16.0 * (double)P.T;
        if (sc > 6.0e9) sc = 6.0e9;
        P.scap = (long long)sc;
    }
    P.nbins = (size_t)P.NC * P.T;
    if (P.nbins > (size_t)0x7fffffff) return fail(BLUR_EINVAL, "too many (chunk, tile) bins");
    const double factor = (cfg && cfg->bin_factor > 0.f) ? cfg->bin_factor : 3.0;
    double cap = factor * (double)P.NC * (double)F + 16.0 * (double)P.T;
    if (cap > 6.0e9) cap = 6.0e9;     // beyond this, overflowing tiles take the exact fallback path
    P.cap = (long long)cap;
    // workspace layout
    size_t o = 0;
    P.o_status = o; o = align256(o + 256);
    P.o_imgs = o; o = align256(o + sizeof(ImgInfo) * (size_t)B);
    P.o_chunks = o; o = align256(o + sizeof(Chunk) * P.chunks.size());
    P.o_ss = o; o = align256(o + sizeof(int) * P.sched_s.size());
    P.o_st = o; o = align256(o + sizeof(float) * P.sched_tau.size());
    P.o_poses = o; o = align256(o + sizeof(PoseRec) * P.poses.size());
    P.o_tables_end = o;
    P.o_key = o; o = align256(o + 16 * (size_t)P.n_key);
    P.o_rec = o; o = align256(o + 16 * REC_F4 * (size_t)P.n_rec);
    P.o_fcol = o; o = align256(o + 48 * (size_t)F);
    P.o_cnt = o; o = align256(o + 4 * P.nbins);
    P.o_off = o; o = align256(o + 8 * (P.nbins + 1));
    P.o_bsum = o; o = align256(o + 8 * ((P.nbins + 1023) / 1024 + 1));
    P.o_ent = o; o = align256(o + 4 * (size_t)P.cap);
    P.o_dkey = o; o = align256(o + 8 * (size_t)P.n_key);
    P.o_part = o; o = align256(o + (P.splits > 1 ? 16 * (size_t)P.splits * B * H * W : 0));
    if (P.soft) {
        P.o_cov = o; o = align256(o + 4 * (size_t)P.n_sub * P.T * (NT / 32));
        P.o_spart = o; o = align256(o + 4 * (size_t)P.ssplits * B * H * W);
        P.o_scnt = o; o = align256(o + 4 * P.nbins);
        P.o_soff = o; o = align256(o + 8 * (P.nbins + 1));
        P.o_sbsum = o; o = align256(o + 8 * ((P.nbins + 1023) / 1024 + 1));
        P.o_sent = o; o = align256(o + 4 * (size_t)P.scap);
    }
    // BLUR_CACHE_VISIBILITY: the soft product cache K8 -> K9 (NEXT-1); the hard path's per-(pixel,
    // sub-frame) winner buffer only for round 1's legacy kernels (the span raster recomputes winners)
    const bool cache = cfg && (cfg->flags & BLUR_CACHE_VISIBILITY) && cfg->solver == 0;
    P.vis = cache && legacy_env();
    P.spz_on = cache && P.soft;
    if (P.vis) { P.o_vis = o; o = align256(o + 2 * (size_t)P.n_sub * P.T * TW * TH); }
    if (P.vis) { P.o_vgl = o; o = align256(o + 16 + 4 * (size_t)P.T * B); }
    if (P.spz_on) { P.o_spz = o; o = align256(o + 4 * (size_t)P.n_sub * P.T * TW * TH); }
    P.total = o;
    return BLUR_OK;
}

Tables make_tables(const Plan &P, void *ws)
{
    char *w = (char *)ws;
    Tables t;
    std::memset(&t, 0, sizeof(t));
    t.status = (int *)(w + P.o_status);
    t.binstat = (long long *)(w + P.o_status + 8);
    t.orient = (double *)(w + P.o_status + 64);
    t.imgs = (const ImgInfo *)(w + P.o_imgs);
    t.chunks = (const Chunk *)(w + P.o_chunks);
    t.sched_s = (const int *)(w + P.o_ss);
    t.sched_tau = (const float *)(w + P.o_st);
    t.poses = (const PoseRec *)(w + P.o_poses);
    t.key = (float4 *)(w + P.o_key);
    t.rec = (float4 *)(w + P.o_rec);
    t.fcol = (float4 *)(w + P.o_fcol);
    t.cnt = (int *)(w + P.o_cnt);
    t.off = (long long *)(w + P.o_off);
    t.bsum = (long long *)(w + P.o_bsum);
    t.entries = (int *)(w + P.o_ent);
    t.cap = P.cap;
    t.dkey = (float2 *)(w + P.o_dkey);
    t.NC = P.NC; t.T = P.T; t.TX = P.TX; t.TY = P.TY;
    t.splits = P.splits;
    t.ssplits = P.ssplits;
    t.part = (float4 *)(w + P.o_part);
    t.B = P.B; t.V = P.V; t.F = P.F; t.H = P.H; t.W = P.W;
    if (P.soft) {
        t.delta = P.delta;
        t.rcut = P.rcut;
        t.rcut_f = P.rcut_f;
        t.soft_exact = P.soft_exact;
        t.covbits = (uint32_t *)(w + P.o_cov);
        t.spart = (float *)(w + P.o_spart);
        t.sb.cnt = (int *)(w + P.o_scnt);
        t.sb.off = (long long *)(w + P.o_soff);
        t.sb.bsum = (long long *)(w + P.o_sbsum);
        t.sb.entries = (int *)(w + P.o_sent);
        t.sb.cap = P.scap;
        t.sb.binstat = (long long *)(w + P.o_status + 24);
        t.sb.sortcap = 16384;   // k_bin.cu SORTCAP_BIG
    }
    if (P.vis) t.vis = (uint16_t *)(w + P.o_vis);
    if (P.vis) { t.vg_count = (int *)(w + P.o_vgl); t.vg_list = (int *)(w + P.o_vgl + 16); }
    if (P.spz_on) t.spz = (float *)(w + P.o_spz);
    t.legacy = legacy_env() ? 1 : 0;
    return t;
}

BinSet hard_bins(const Tables &t)
{
    BinSet b;
    b.cnt = t.cnt;
    b.off = t.off;
    b.bsum = t.bsum;
    b.entries = t.entries;
    b.cap = t.cap;
    b.binstat = t.binstat;
#ifdef BR_SORT_HARD
    b.sortcap = SORTCAP;
#else
    b.sortcap = 0;      // not sorted: the raster z-buffer breaks depth ties by face index itself
#endif
    return b;
}

int upload_tables(const Plan &P, void *ws, cudaStream_t st)
{
    std::vector<char> h(P.o_tables_end - P.o_imgs, 0);
    auto put = [&](size_t off, const void *src, size_t n) {
        if (n) std::memcpy(h.data() + (off - P.o_imgs), src, n);
    };
    put(P.o_imgs, P.imgs.data(), sizeof(ImgInfo) * P.imgs.size());
    put(P.o_chunks, P.chunks.data(), sizeof(Chunk) * P.chunks.size());
    put(P.o_ss, P.sched_s.data(), sizeof(int) * P.sched_s.size());
    put(P.o_st, P.sched_tau.data(), sizeof(float) * P.sched_tau.size());
    put(P.o_poses, P.poses.data(), sizeof(PoseRec) * P.poses.size());
    cudaError_t e = cudaMemcpyAsync((char *)ws + P.o_imgs, h.data(), h.size(), cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return fail(BLUR_ECUDA, std::string("table upload: ") + cudaGetErrorString(e));
    return BLUR_OK;
}

int cuda_check(cudaError_t e, const char *what)
{
    if (e != cudaSuccess) return fail(BLUR_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
    return BLUR_OK;
}

// Raster kernels of the fast solver: BLURRAST_RASTER=span selects k_span.cu's span raster (A/B while it
// is tuned), otherwise round 1's footprint-mask kernels (k_raster.cu)
bool legacy_env()
{
    const char *s = std::getenv("BLURRAST_RASTER");
    return !(s && std::strcmp(s, "span") == 0);
}

bool check_env()
{
    const char *s = std::getenv("BLURRAST_CHECK");
    return s && s[0] == '1';
}

int status_to_code(int st)
{
    if (st & BLUR_ST_EINTERNAL) return fail(BLUR_ECUDA, "internal consistency check failed");
    if (st & BLUR_ST_EINVAL) return fail(BLUR_EINVAL, "a face index is out of range [0, V)");
    if (st & BLUR_ST_EBEHIND) return fail(BLUR_EBEHIND, "a vertex is at or behind the near plane");
    if (st & BLUR_ST_EOVERFLOW) return fail(BLUR_EOVERFLOW, "bin capacity exceeded (exact slow path used)");
    return BLUR_OK;
}

int sync_status(void *ws, const Plan &P, cudaStream_t st)
{
    int h = 0;
    int r = cuda_check(cudaMemcpyAsync(&h, (char *)ws + P.o_status, sizeof(int), cudaMemcpyDeviceToHost, st), "status read");
    if (r) return r;
    r = cuda_check(cudaStreamSynchronize(st), "stream sync");
    if (r) return r;
    return status_to_code(h);
}

int prepare(const float *verts, int V, const int32_t *faces, int F, const float *colors, const blur_motion *m,
            const blur_camera *cams, int B, int H, int W, const int32_t *sub_range, const blur_config *cfg,
            void *ws, size_t ws_bytes, cudaStream_t st, bool do_setup, Plan &P, Tables &t)
{
    int r = make_plan(V, F, B, H, W, m, cams, sub_range, cfg, P);
    if (r) return r;
    if (B > 0 && (!verts && V > 0)) return fail(BLUR_EINVAL, "verts is NULL");
    if (F > 0 && (!faces || !colors)) return fail(BLUR_EINVAL, "faces or colors is NULL");
    if (!ws) return fail(BLUR_EINVAL, "workspace is NULL");
    if (ws_bytes < P.total)
        return fail(BLUR_ENOMEM, "workspace too small: need " + std::to_string(P.total) + " bytes");
    t = make_tables(P, ws);
    t.solver = cfg ? cfg->solver : 0;
    if (t.solver < 0 || t.solver > 2) return fail(BLUR_EINVAL, "solver must be 0, 1 or 2");
    if (!do_setup) return BLUR_OK;
    r = cuda_check(cudaMemsetAsync(t.status, 0, sizeof(int), st), "status clear");
    if (r) return r;
    if (!(cfg && (cfg->flags & BLUR_TABLES_RESIDENT))) {   // host tables (pageable copy): not capturable
        r = upload_tables(P, ws, st);
        if (r) return r;
    }
    {
        Nvtx n("K1-K2 setup");
        r = cuda_check(launch_setup(t, verts, faces, colors, P.maxS, st), "setup kernels");
        if (r) return r;
    }
    // (the soft bins are built after K4: their sort skips the tiles K4 found fully covered)
    Nvtx n("K3 binning");
    return cuda_check(launch_binning(t, hard_bins(t), 0.f, st), "binning kernels");
}

}  // namespace

namespace br {
void set_last_error(const std::string &msg) { g_err = msg; }
void clear_last_error() { g_err.clear(); }
}  // namespace br

extern "C" {

const char *blur_last_error(void) { return g_err.c_str(); }

int blur_abi_version(void) { return 2; }

size_t blur_workspace_bytes(int V, int F, int B, int H, int W, const blur_motion *motions,
                            const blur_camera *cams, const int32_t *sub_range, const blur_config *cfg)
{
    g_err.clear();
    Plan P;
    if (B > 0 && !cams) { fail(BLUR_EINVAL, "cams is NULL"); return 0; }
    if (make_plan(V, F, B, H, W, motions, cams, sub_range, cfg, P)) return 0;
    return P.total;
}

int blur_render_fwd(const float *verts, int V, const int32_t *faces, int F, const float *colors,
                    const blur_motion *motions, const blur_camera *cams, int B, int H, int W,
                    const int32_t *sub_range, float *out_rgba, int32_t *ids, int ids_subframe,
                    const blur_config *cfg, void *ws, size_t ws_bytes, blur_stream_t stream)
{
    Nvtx range("blur_render_fwd");
    g_err.clear();
    cudaStream_t st = (cudaStream_t)stream;
    if (B > 0 && !cams) return fail(BLUR_EINVAL, "cams is NULL");
    if (B > 0 && !out_rgba) return fail(BLUR_EINVAL, "out_rgba is NULL");
    Plan P;
    Tables t;
    int r = prepare(verts, V, faces, F, colors, motions, cams, B, H, W, sub_range, cfg, ws, ws_bytes, st, true, P, t);
    if (r) return r;
    if (cfg && cfg->raster_events[0]) cudaEventRecord((cudaEvent_t)cfg->raster_events[0], st);
    {
        Nvtx n("K4 raster fwd");
        r = cuda_check(launch_raster_fwd(t, out_rgba, ids, ids_subframe, cfg ? cfg->census : nullptr, st), "raster fwd");
        if (r) return r;
    }
    if (P.splits > 1) {
        r = cuda_check(launch_split_reduce(t, out_rgba, st), "split reduce");
        if (r) return r;
    }
    if (cfg && cfg->raster_events[1]) cudaEventRecord((cudaEvent_t)cfg->raster_events[1], st);
    if (P.soft) {   // NEXT-1: background alpha of the uncovered (pixel, sub-frame) pairs K4 recorded
        Nvtx n("K8 soft fwd");
        r = cuda_check(launch_binning(t, t.sb, P.rcut, st), "soft binning kernels");
        if (r) return r;
        if (cfg->soft_events[0]) cudaEventRecord((cudaEvent_t)cfg->soft_events[0], st);
        r = cuda_check(launch_soft_fwd(t, out_rgba, cfg->census, st), "soft fwd");
        if (r) return r;
        if (cfg->soft_events[1]) cudaEventRecord((cudaEvent_t)cfg->soft_events[1], st);
    }
    if (check_env()) return sync_status(ws, P, st);
    return BLUR_OK;
}

int blur_render_bwd(const float *verts, int V, const int32_t *faces, int F, const float *colors,
                    const blur_motion *motions, const blur_camera *cams, int B, int H, int W,
                    const int32_t *sub_range, const float *grad_rgba, float *grad_verts, float *grad_colors,
                    const blur_config *cfg, void *ws, size_t ws_bytes, blur_stream_t stream)
{
    Nvtx range("blur_render_bwd");
    g_err.clear();
    cudaStream_t st = (cudaStream_t)stream;
    if (B > 0 && !cams) return fail(BLUR_EINVAL, "cams is NULL");
    if (V > 0 && (!grad_verts || !grad_colors)) return fail(BLUR_EINVAL, "gradient outputs are NULL");
    if (B > 0 && !grad_rgba) return fail(BLUR_EINVAL, "grad_rgba is NULL");
    const bool reuse = cfg && (cfg->flags & BLUR_REUSE_SETUP);
    Plan P;
    Tables t;
    int r = prepare(verts, V, faces, F, colors, motions, cams, B, H, W, sub_range, cfg, ws, ws_bytes, st, !reuse, P, t);
    if (r) return r;
    if (V > 0) {
        r = cuda_check(cudaMemsetAsync(grad_colors, 0, sizeof(float) * 3 * (size_t)V, st), "grad clear");
        if (r) return r;
    }
    if (P.n_key) {
        r = cuda_check(cudaMemsetAsync(t.dkey, 0, 8 * (size_t)P.n_key, st), "dkey clear");
        if (r) return r;
    }
    if (!reuse) {   // the visibility and soft-product buffers are only valid right after the forward
        t.vis = nullptr;
        t.spz = nullptr;
    }
    if (P.soft && !reuse) {   // coverage of every (pixel, sub-frame) for the soft term (no image written)
        r = cuda_check(launch_raster_fwd(t, nullptr, nullptr, -1, nullptr, st), "coverage pass");
        if (r) return r;
        r = cuda_check(launch_binning(t, t.sb, P.rcut, st), "soft binning kernels");
        if (r) return r;
    }
    if (cfg && cfg->raster_events[0]) cudaEventRecord((cudaEvent_t)cfg->raster_events[0], st);
    {
        Nvtx n("K6 raster bwd");
        r = cuda_check(launch_raster_bwd(t, grad_rgba, grad_colors, st), "raster bwd");
        if (r) return r;
    }
    if (cfg && cfg->raster_events[1]) cudaEventRecord((cudaEvent_t)cfg->raster_events[1], st);
    if (P.soft) {
        Nvtx n("K9 soft bwd");
        if (cfg->soft_events[0]) cudaEventRecord((cudaEvent_t)cfg->soft_events[0], st);
        r = cuda_check(launch_soft_bwd(t, grad_rgba, st), "soft bwd");
        if (r) return r;
        if (cfg->soft_events[1]) cudaEventRecord((cudaEvent_t)cfg->soft_events[1], st);
    }
    Nvtx n("K7 vertex chain");
    r = cuda_check(launch_vertex_chain(t, grad_verts, st), "vertex chain");
    if (r) return r;
    if (check_env()) return sync_status(ws, P, st);
    return BLUR_OK;
}

int blur_l2_loss_grad(const float *out, const float *target, int64_t n, int64_t n_norm, float *loss, float *grad,
                      blur_stream_t stream)
{
    Nvtx range("blur_l2_loss_grad");
    g_err.clear();
    if (n < 0) return fail(BLUR_EINVAL, "n < 0");
    if (!loss || (n > 0 && (!out || !target || !grad))) return fail(BLUR_EINVAL, "NULL pointer");
    if ((((uintptr_t)out) | ((uintptr_t)target) | ((uintptr_t)grad)) & 15)
        return fail(BLUR_EINVAL, "out/target/grad must be 16-byte aligned");
    return cuda_check(launch_l2(out, target, n, n_norm, loss, grad, (cudaStream_t)stream), "l2 loss");
}

int blur_read_status(void *ws, blur_stream_t stream, int32_t *status_out)
{
    g_err.clear();
    if (!ws || !status_out) return fail(BLUR_EINVAL, "NULL pointer");
    cudaStream_t st = (cudaStream_t)stream;
    int h = 0;
    int r = cuda_check(cudaMemcpyAsync(&h, ws, sizeof(int), cudaMemcpyDeviceToHost, st), "status read");
    if (r) return r;
    r = cuda_check(cudaStreamSynchronize(st), "stream sync");
    if (r) return r;
    *status_out = h;
    return cuda_check(cudaMemsetAsync(ws, 0, sizeof(int), st), "status clear");
}

int blur_read_bins(void *ws, blur_stream_t stream, long long *needed, long long *capacity)
{
    g_err.clear();
    if (!ws || !needed || !capacity) return fail(BLUR_EINVAL, "NULL pointer");
    cudaStream_t st = (cudaStream_t)stream;
    long long h[2] = {0, 0};
    int r = cuda_check(cudaMemcpyAsync(h, (char *)ws + 8, sizeof(h), cudaMemcpyDeviceToHost, st), "bins read");
    if (r) return r;
    r = cuda_check(cudaStreamSynchronize(st), "stream sync");
    if (r) return r;
    *needed = h[0];
    *capacity = h[1];
    return BLUR_OK;
}

int blur_read_soft_bins(void *ws, blur_stream_t stream, long long *needed, long long *capacity)
{
    g_err.clear();
    if (!ws || !needed || !capacity) return fail(BLUR_EINVAL, "NULL pointer");
    cudaStream_t st = (cudaStream_t)stream;
    long long h[2] = {0, 0};
    int r = cuda_check(cudaMemcpyAsync(h, (char *)ws + 24, sizeof(h), cudaMemcpyDeviceToHost, st), "bins read");
    if (r) return r;
    r = cuda_check(cudaStreamSynchronize(st), "stream sync");
    if (r) return r;
    *needed = h[0];
    *capacity = h[1];
    return BLUR_OK;
}

int blur_ffma_probe(int ctas, int iters, float *sink, double *flops, blur_stream_t stream)
{
    g_err.clear();
    if (ctas < 1 || iters < 1 || !sink || !flops) return fail(BLUR_EINVAL, "bad probe arguments");
    *flops = 2.0 * 16.0 * 8.0 * (double)iters * 256.0 * (double)ctas;
    return cuda_check(launch_ffma_probe(ctas, iters, sink, (cudaStream_t)stream), "ffma probe");
}

}  // extern "C"
