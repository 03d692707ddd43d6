/*
 * oracle.c -- plain, slow, fp64 CPU oracle for the motion-blur hot path of
 * arxiv 2602.07860 ("fast barycentric solver for ultra-fast motion blur").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It
 * shares no code, header, table or helper with the CUDA path
 * (paper_2602_07860_b200/csrc); neither side includes or links the other.
 *
 * Citations: "P:L###" is a line of /root/reference/PAPER.md (Eq.n numbered by
 * \begin{equation} order, appendix A1..A37), "S:L###" a line of SPEC.md.
 * Readings of passages where the paper is silent/ambiguous are the "Q#"
 * entries of DESIGN.md (same numbering as SURVEY.md 8(c)).
 *
 * What is computed:
 *   for every image b and sub-frame k of the schedule (Q1):
 *     keyframes: exact rigid pose at t = s/S (A30/A31 generalised, Q2-Q4),
 *                projected with A34 (camera frame Q5) -> NDC x, y and view z
 *     sub-frame geometry: screen-space lerp of keyframes s_k, s_k+1 at tau_k
 *                (Eq.5-6)
 *     per pixel centre (Q9), per face in index order: textbook solve
 *                w = F^-1 p = adj(F) p / det F (Eq.3, Eq.7; A8, A9),
 *                skip |det| <= EPS_D (Q8), covered iff all w_i >= 0 (Q7),
 *                z = sum w_i z_i (Q6), strict less-than z-buffer (lowest index
 *                wins exact ties, Q7)
 *     value: covered -> (sum w_i c_i, 1) (Eq.9); else (0,0,0,0) (Q10)
 *     blurred image = uniform mean over the N sub-frames (Q1)
 *   backward (frozen winner Q11): dL/dc_i += w_i G/N;
 *     dL/dv_i(tau) = sum_j (G.c_j/N) dw_j/dv_i with dw/dv_i = -w_i dw/dp,
 *     split (1-tau), tau onto keyframes, chained through A34, the camera
 *     rotation and the pose to world vertices.
 *   fast-solver cross-check: Eq.8 with the coefficients A11-A16 transcribed
 *     literally evaluated for every covered pair.
 *
 *   soft background coverage (NEXT-1; opts.delta > 0): a pixel with no covering face at a
 *     sub-frame gets RGB 0 and alpha A_i(t) = 1 - prod_j (1 - A_i^j(t)) over all faces valid at
 *     tau (Eq.15), A = exp(-d/delta) (Eq.10, A20), d from the closest point on the keyframe
 *     triangle F(X) (Eq.13, A17-A18) mapped to F(tau) (Eq.14); backward with w^* frozen.
 *
 * Modes: brute (all pixels x all faces) and binned (per face, pixels inside
 * the face's bounding box -- an exact cull for this coverage rule; the per
 * pixel arithmetic and the face order are unchanged, so the two modes are
 * bit-identical; pinned by tests/test_oracle_pins.py).
 */
#define _GNU_SOURCE
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OM_STATIC 0
#define OM_TRANSLATE 1
#define OM_ROTATE 2
#define OM_PARABOLIC 3
#define OM_GLOBAL_INCLUSIVE 0
#define OM_PAPER_SEGMENTED 1

static const double EPS_D = 1e-12;      /* Q8: degenerate if |det F| <= 1e-12 NDC^2 */

typedef struct {
    int V, F, B, H, W;
    const double *verts;   /* V*3 world positions */
    const int *faces;      /* F*3 */
    const double *colors;  /* V*3 */
    const double *cams;    /* B*11: eye target up half_fov z_near */
    const int *kind;       /* B */
    const double *vec;     /* B*3 */
    const double *angle;   /* B */
    const double *pivot;   /* B*3 */
    const int *n_sub;      /* B */
    const int *n_seg;      /* B */
    const int *rule;       /* B */
    const int *sub_range;  /* B*2 [k0,k1) or NULL */
} om_scene;

typedef struct {
    int mode;              /* 0 brute, 1 binned */
    int threads;           /* 0 = OpenMP default */
    int check_fast;        /* evaluate A11-A16 literally for every covered pair */
    double eps_amb;        /* Q16 edge-distance epsilon (NDC); <= 0 disables ambiguity analysis */
    double amb_val_tol;    /* Q16 shaded-value change threshold (1e-5) */
    double amb_z_rel;      /* Q16 relative depth-tie tolerance (1e-6) */
    int npix;              /* >0: evaluate only the listed pixels (pixel-list mode) */
    const int *pix;        /* npix*3: (b, row, col) */
    double delta;          /* soft background bandwidth (NDC^2, Eq.10); 0 = hard coverage only */
    int soft_exact;        /* 1: Eq.12 (closest point on F(tau) itself) instead of Eq.13's F(X) */
} om_opts;

/* --------------------------------------------------------------- schedule */

/* Q1 reading of P:L235 / P:L280 / P:L1256.
 * GLOBAL_INCLUSIVE: t_k = k/(N-1) (N=1 -> 0.5); s_k = min(floor(t_k S), S-1); tau_k = t_k S - s_k,
 *   evaluated in integer arithmetic: s = min(kS div (N-1), S-1), tau = (kS - s(N-1))/(N-1).
 * PAPER_SEGMENTED: S | N, K = N/S, s = k div K, tau = (k mod K)/(K-1) (K=1 -> 0.5). */
int om_schedule(int N, int S, int rule, int *s_out, double *tau_out)
{
    if (N < 1 || S < 1) return -1;
    if (rule == OM_PAPER_SEGMENTED) {
        if (N % S) return -1;
        int K = N / S;
        for (int k = 0; k < N; ++k) {
            s_out[k] = k / K;
            tau_out[k] = (K == 1) ? 0.5 : (double)(k % K) / (double)(K - 1);
        }
        return 0;
    }
    if (rule != OM_GLOBAL_INCLUSIVE) return -1;
    if (N == 1) {
        int s = S / 2;               /* t = 0.5 -> t*S = S/2 */
        if (s > S - 1) s = S - 1;
        s_out[0] = s;
        tau_out[0] = 0.5 * S - s;
        return 0;
    }
    for (int k = 0; k < N; ++k) {
        long num = (long)k * S;
        long s = num / (N - 1);
        if (s > S - 1) s = S - 1;
        s_out[k] = (int)s;
        tau_out[k] = (double)(num - s * (N - 1)) / (double)(N - 1);
    }
    return 0;
}

/* Segment count of image b (Q24): n_seg as given, or for n_seg == 0 the paper's segmentation rule --
 * one linear segment for translation / static, ceil(12 turns - 1e-6) for rotation (12 per full turn,
 * P:L277; the 1e-6 keeps an fp32 angle of a whole number of turns from adding a segment), at least one. */
int om_segments(const om_scene *sc, int b)
{
    int S = sc->n_seg[b];
    if (S != 0) return S;
    if (sc->kind[b] == OM_ROTATE || sc->kind[b] == OM_PARABOLIC) {
        double turns = fabs(sc->angle[b]) / (2.0 * M_PI);
        int s12 = (int)ceil(12.0 * turns - 1e-6);   /* float angles of whole turns stay whole */
        return s12 < 1 ? 1 : s12;
    }
    return 1;
}

/* --------------------------------------------------------------- pose + projection */

static void cross3(const double a[3], const double b[3], double o[3])
{
    o[0] = a[1] * b[2] - a[2] * b[1];
    o[1] = a[2] * b[0] - a[0] * b[2];
    o[2] = a[0] * b[1] - a[1] * b[0];
}
static double dot3(const double a[3], const double b[3]) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
static void normalize3(double a[3])
{
    double n = sqrt(dot3(a, a));
    a[0] /= n; a[1] /= n; a[2] /= n;
}

/* Right-handed Rodrigues rotation R(axis, theta) = I + sin K + (1-cos) K^2 (Q4; agrees with
 * the rotation written out in P:L1615-1617). */
static void rodrigues(const double ax[3], double th, double R[9])
{
    double a[3] = {ax[0], ax[1], ax[2]};
    normalize3(a);
    double K[9] = {0, -a[2], a[1], a[2], 0, -a[0], -a[1], a[0], 0};
    double K2[9];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double s = 0;
            for (int l = 0; l < 3; ++l) s += K[i * 3 + l] * K[l * 3 + j];
            K2[i * 3 + j] = s;
        }
    double sn = sin(th), cs = 1.0 - cos(th);
    for (int i = 0; i < 9; ++i) R[i] = ((i % 4) == 0 ? 1.0 : 0.0) + sn * K[i] + cs * K2[i];
}

/* Rigid pose at exposure time t, written P(t) = R (P0 - c) + c + T for every kind:
 *  translate (A30 P:L1417-1424 generalised, Q2): R = I, T = (t - 0.5) vec
 *  rotate    (A31 P:L1430-1432 generalised, Q3/Q4): R = R(a, Theta t), c = pivot
 *  parabolic (A35-A37 P:L1613-1629 generalised): R = R(a, Theta t), c = pivot,
 *            T = (s, -4 s^2 + 0.5, s) with s = 0.5 - t (the paper's case: a = y, Theta = pi, c = 0) */
static void pose_rct(const om_scene *sc, int b, double t, double R[9], double c[3], double T[3])
{
    int kind = sc->kind[b];
    const double *vec = sc->vec + 3 * b, *piv = sc->pivot + 3 * b;
    for (int i = 0; i < 9; ++i) R[i] = (i % 4) == 0 ? 1.0 : 0.0;
    c[0] = c[1] = c[2] = 0.0;
    T[0] = T[1] = T[2] = 0.0;
    if (kind == OM_TRANSLATE) {
        for (int i = 0; i < 3; ++i) T[i] = (t - 0.5) * vec[i];
    } else if (kind == OM_ROTATE || kind == OM_PARABOLIC) {
        rodrigues(vec, sc->angle[b] * t, R);
        for (int i = 0; i < 3; ++i) c[i] = piv[i];
        if (kind == OM_PARABOLIC) {
            double s = 0.5 - t;
            T[0] = s;
            T[1] = -4.0 * s * s + 0.5;
            T[2] = s;
        }
    }
}

/* the rotation part only (for the backward chain) */
static void pose_rt(const om_scene *sc, int b, double t, double R[9], double tr[3])
{
    double c[3], T[3];
    pose_rct(sc, b, t, R, c, T);
    (void)tr;
}

/* Camera frame: forward f = normalize(target - eye), right r = normalize(f x up), up' = r x f.
 * View coordinates Q = (r.(P-E), up'.(P-E), f.(P-E)) (Q5). */
static void cam_frame(const double *cam, double Rc[9])
{
    double f[3] = {cam[3] - cam[0], cam[4] - cam[1], cam[5] - cam[2]};
    normalize3(f);
    double r[3], u[3];
    cross3(f, cam + 6, r);
    normalize3(r);
    cross3(r, f, u);
    for (int i = 0; i < 3; ++i) { Rc[i] = r[i]; Rc[3 + i] = u[i]; Rc[6 + i] = f[i]; }
}

/* Keyframes of image b: for s = 0..S, vertex v -> (x_ndc, y_ndc, z_view) by A34:
 * x = Qx / (Qz tan(alpha)), y = Qy / (Qz tan(alpha)), z = Qz.  valid = Qz > z_near.
 * Optionally returns the view coordinates Q (for the backward chain). */
int om_keyframes(const om_scene *sc, int b, double *key, unsigned char *valid, double *Qout)
{
    int S = om_segments(sc, b), V = sc->V;
    const double *cam = sc->cams + 11 * b;
    double Rc[9];
    cam_frame(cam, Rc);
    double ta = tan(cam[9]);
    int bad = 0;
    for (int s = 0; s <= S; ++s) {
        double R[9], c[3], T[3];
        pose_rct(sc, b, (double)s / (double)S, R, c, T);
        for (int v = 0; v < V; ++v) {
            const double *P0 = sc->verts + 3 * v;
            double P[3], d[3], Q[3];
            double q[3] = {P0[0] - c[0], P0[1] - c[1], P0[2] - c[2]};
            for (int i = 0; i < 3; ++i)
                P[i] = R[i * 3] * q[0] + R[i * 3 + 1] * q[1] + R[i * 3 + 2] * q[2] + c[i] + T[i];
            for (int i = 0; i < 3; ++i) d[i] = P[i] - cam[i];
            for (int i = 0; i < 3; ++i) Q[i] = Rc[i * 3] * d[0] + Rc[i * 3 + 1] * d[1] + Rc[i * 3 + 2] * d[2];
            size_t o = ((size_t)s * V + v);
            key[3 * o + 0] = Q[0] / (Q[2] * ta);
            key[3 * o + 1] = Q[1] / (Q[2] * ta);
            key[3 * o + 2] = Q[2];
            valid[o] = Q[2] > cam[10];
            if (!valid[o]) bad = 1;
            if (Qout) { Qout[3 * o] = Q[0]; Qout[3 * o + 1] = Q[1]; Qout[3 * o + 2] = Q[2]; }
        }
    }
    return bad;
}

/* --------------------------------------------------------------- barycentric solvers */

/* Textbook solve (Eq.3, Eq.7): w = adj(F) p / det(F), det by A8, adj by A9
 * (P:L989-999), p = (u, v, 1).  Returns 0 if |det| <= EPS_D (Q8). */
int om_bary_textbook(const double x[3], const double y[3], double u, double v, double w[3], double *det_out)
{
    double det = x[0] * (y[1] - y[2]) - x[1] * (y[0] - y[2]) + x[2] * (y[0] - y[1]);
    *det_out = det;
    if (!(fabs(det) > EPS_D)) return 0;
    double n0 = (y[1] - y[2]) * u + (x[2] - x[1]) * v + (x[1] * y[2] - x[2] * y[1]);
    double n1 = (y[2] - y[0]) * u + (x[0] - x[2]) * v + (x[2] * y[0] - x[0] * y[2]);
    double n2 = (y[0] - y[1]) * u + (x[1] - x[0]) * v + (x[0] * y[1] - x[1] * y[0]);
    w[0] = n0 / det;
    w[1] = n1 / det;
    w[2] = n2 / det;
    return 1;
}

/* The paper's fast-solver coefficients, transcribed literally from A11-A16.
 * Arguments: keyframe triangles F(0) = (X0, Y0) and F(1) = (X1, Y1), pixel (u, v).
 * w(t) = (A1 t^2 + A2 t + A3) / (a1 t^2 + a2 t + a3)  (Eq.8). */
void om_fast_coeffs(const double X0[3], const double Y0[3], const double X1[3], const double Y1[3],
                    double u, double v, double A1[3], double A2[3], double A3[3], double a[3])
{
#define x0_0 X0[0]
#define x1_0 X0[1]
#define x2_0 X0[2]
#define y0_0 Y0[0]
#define y1_0 Y0[1]
#define y2_0 Y0[2]
#define x0_1 X1[0]
#define x1_1 X1[1]
#define x2_1 X1[2]
#define y0_1 Y1[0]
#define y1_1 Y1[1]
#define y2_1 Y1[2]
    /* A11 */
    A1[0] = -(x2_0 - x2_1) * (y1_0 - y1_1) + (x1_0 - x1_1) * (y2_0 - y2_1);
    A1[1] = ((x2_0 - x2_1) * (y0_0 - y0_1) - (x0_0 - x0_1) * (y2_0 - y2_1));
    A1[2] = (-((x1_0 - x1_1) * (y0_0 - y0_1)) + (x0_0 - x0_1) * (y1_0 - y1_1));
    /* A12 */
    A2[0] = u * (-y1_0 + y2_0 + y1_1 - y2_1) + v * (x1_0 - x2_0 - x1_1 + x2_1) +
            (y2_0 * x1_1 - y1_0 * x2_1 + x2_0 * (2 * y1_0 - y1_1) + x1_0 * (-2 * y2_0 + y2_1));
    A2[1] = u * (y0_0 - y2_0 - y0_1 + y2_1) + v * (-x0_0 + x2_0 + x0_1 - x2_1) +
            (-(y2_0 * x0_1) + y0_0 * x2_1 + x2_0 * (-2 * y0_0 + y0_1) + x0_0 * (2 * y2_0 - y2_1));
    A2[2] = u * (-y0_0 + y1_0 + y0_1 - y1_1) + v * (x0_0 - x1_0 - x0_1 + x1_1) +
            (y1_0 * x0_1 - y0_0 * x1_1 + x1_0 * (2 * y0_0 - y0_1) + x0_0 * (-2 * y1_0 + y1_1));
    /* A13 */
    A3[0] = u * (y1_0 - y2_0) + v * (-x1_0 + x2_0) + (-(x2_0 * y1_0) + x1_0 * y2_0);
    A3[1] = u * (-y0_0 + y2_0) + v * (x0_0 - x2_0) + (x2_0 * y0_0 - x0_0 * y2_0);
    A3[2] = u * (y0_0 - y1_0) + v * (-x0_0 + x1_0) + (-(x1_0 * y0_0) + x0_0 * y1_0);
    /* A14 */
    a[0] = -(y1_0 * x0_1) + y2_0 * x0_1 - y2_0 * x1_1 + y0_0 * (x1_1 - x2_1) + y1_0 * x2_1 - x1_1 * y0_1 +
           x2_1 * y0_1 + x0_1 * y1_1 - x2_1 * y1_1 + x2_0 * (y0_0 - y1_0 - y0_1 + y1_1) +
           x1_0 * (-y0_0 + y2_0 + y0_1 - y2_1) - x0_1 * y2_1 + x1_1 * y2_1 + x0_0 * (y1_0 - y2_0 - y1_1 + y2_1);
    /* A15 */
    a[1] = y1_0 * x0_1 - y2_0 * x0_1 + y2_0 * x1_1 - y1_0 * x2_1 + y0_0 * (-x1_1 + x2_1) +
           x2_0 * (-2 * y0_0 + 2 * y1_0 + y0_1 - y1_1) + x0_0 * (-2 * y1_0 + 2 * y2_0 + y1_1 - y2_1) +
           x1_0 * (2 * y0_0 - 2 * y2_0 - y0_1 + y2_1);
    /* A16 */
    a[2] = x2_0 * (y0_0 - y1_0) + x0_0 * (y1_0 - y2_0) + x1_0 * (-y0_0 + y2_0);
#undef x0_0
#undef x1_0
#undef x2_0
#undef y0_0
#undef y1_0
#undef y2_0
#undef x0_1
#undef x1_1
#undef x2_1
#undef y0_1
#undef y1_1
#undef y2_1
}

/* Eq.8 evaluated at t.  Returns 0 if |denominator| <= EPS_D. */
int om_fast_eval(const double X0[3], const double Y0[3], const double X1[3], const double Y1[3],
                 double u, double v, double t, double w[3], double *den_out)
{
    double A1[3], A2[3], A3[3], a[3];
    om_fast_coeffs(X0, Y0, X1, Y1, u, v, A1, A2, A3, a);
    double den = a[0] * t * t + a[1] * t + a[2];
    *den_out = den;
    if (!(fabs(den) > EPS_D)) return 0;
    for (int i = 0; i < 3; ++i) w[i] = (A1[i] * t * t + A2[i] * t + A3[i]) / den;
    return 1;
}

/* --------------------------------------------------------------- soft background coverage (NEXT-1) */

/* Closest point of the triangle (x, y) to the point (pu, pv), as weights (appendix "Euclidean
 * Distance Approximation", A17-A18):
 *   if the point is inside (all barycentric weights w >= 0) the weights are w itself;
 *   otherwise, for the edges v0v1, v1v2, v2v0 in this order, the projection parameter
 *     t = ((u - x_i)(x_j - x_i) + (v - y_i)(y_j - y_i)) / ((x_j - x_i)^2 + (y_j - y_i)^2)   (A17)
 *   gives w'_i = 1 - t, w'_j = t for 0 <= t <= 1, vertex i for t < 0, vertex j for t > 1 (A18
 *   text), and the edge candidate with the smallest squared distance is taken (first
 *   in edge order on exact ties; a zero-length edge is its vertex i -- reading Q19).
 * w_in: barycentric weights of the point w.r.t. this triangle (used for the inside test); may be
 * NULL (then the inside test is skipped).  Outputs: what (the chosen weights), dist2 (its squared
 * distance in this triangle's plane); cand[9]/cd[3] (optional) the three edge candidates and their
 * squared distances (for the ambiguity analysis).  Returns the chosen edge (0..2) or -1 (inside). */
int om_closest_w(const double x[3], const double y[3], double pu, double pv, const double *w_in,
                 double what[3], double *dist2, double *cand, double *cd)
{
    if (w_in && w_in[0] >= 0.0 && w_in[1] >= 0.0 && w_in[2] >= 0.0) {
        for (int i = 0; i < 3; ++i) what[i] = w_in[i];
        *dist2 = 0.0;
        if (cand) for (int e = 0; e < 3; ++e) { cd[e] = 0.0; for (int i = 0; i < 3; ++i) cand[3 * e + i] = w_in[i]; }
        return -1;
    }
    int best = -1;
    double bestd = INFINITY;
    for (int e = 0; e < 3; ++e) {
        int i = e, j = (e + 1) % 3;
        double ex = x[j] - x[i], ey = y[j] - y[i];
        double l2 = ex * ex + ey * ey;
        double t = l2 > 0.0 ? ((pu - x[i]) * ex + (pv - y[i]) * ey) / l2 : 0.0;
        double wc[3] = {0.0, 0.0, 0.0};
        if (t < 0.0) {
            wc[i] = 1.0;
        } else if (t > 1.0) {
            wc[j] = 1.0;
        } else {
            wc[i] = 1.0 - t;
            wc[j] = t;
        }
        double qx = wc[0] * x[0] + wc[1] * x[1] + wc[2] * x[2];
        double qy = wc[0] * y[0] + wc[1] * y[1] + wc[2] * y[2];
        double d = (pu - qx) * (pu - qx) + (pv - qy) * (pv - qy);
        if (cand) { cd[e] = d; for (int q = 0; q < 3; ++q) cand[3 * e + q] = wc[q]; }
        if (d < bestd) {
            bestd = d;
            best = e;
            for (int q = 0; q < 3; ++q) what[q] = wc[q];
        }
    }
    *dist2 = bestd;
    return best;
}

/* One (pixel, face, sub-frame) background term (Eq.10-14).
 * Keyframe triangles F(0) = (X0, Y0), F(1) = (X1, Y1) of the segment, segment time tau, pixel
 * (u, v), bandwidth delta (NDC^2; Q9).  Steps, in the paper's order:
 *   F(tau) = (1 - tau) F(0) + tau F(1) (Eq.5-6); w(tau) = F(tau)^-1 p (Eq.3, textbook solve);
 *   X = 0 if tau <= 0.5 else 1 (Eq.13), or F(X) = F(tau) itself when exact != 0 (Eq.12);
 *   p' = F(X) w(tau); w^* = closest-point weights of p' on F(X) (A17-A18, om_closest_w);
 *   d = || F(tau) w(tau) - F(tau) w^* ||^2 = || p - F(tau) w^* ||^2 (Eq.14);
 *   A = exp(-d / delta) (Eq.10 with the exponential kernel, A20).
 * Outputs A, d, what (w^*), pstar = F(tau) w^* (2), and, when amb != NULL, amb[0] = the largest
 * |A' - A| over the edge candidates that a move of p' by eps NDC could make the closest one
 * (Q20: |d_c - d_e| <= 2 eps |q_c - q_e| + 1e-6 max(d_c, d_e)).  Returns 0 if F(tau) is
 * degenerate (Q8: the face is skipped for this sub-frame), else 1. */
int om_soft_pair(const double X0[3], const double Y0[3], const double X1[3], const double Y1[3], double tau,
                 double u, double v, double delta, int exact, double eps, double *A, double *d, double what[3],
                 double pstar[2], double *amb)
{
    double xt[3], yt[3], w[3], det;
    for (int i = 0; i < 3; ++i) {
        xt[i] = (1.0 - tau) * X0[i] + tau * X1[i];
        yt[i] = (1.0 - tau) * Y0[i] + tau * Y1[i];
    }
    if (!om_bary_textbook(xt, yt, u, v, w, &det)) return 0;
    const double *xk = exact ? xt : (tau <= 0.5 ? X0 : X1);
    const double *yk = exact ? yt : (tau <= 0.5 ? Y0 : Y1);
    double pu = w[0] * xk[0] + w[1] * xk[1] + w[2] * xk[2];
    double pv = w[0] * yk[0] + w[1] * yk[1] + w[2] * yk[2];
    double cand[9], cd[3], dX;
    int e = om_closest_w(xk, yk, pu, pv, w, what, &dX, cand, cd);
    pstar[0] = what[0] * xt[0] + what[1] * xt[1] + what[2] * xt[2];
    pstar[1] = what[0] * yt[0] + what[1] * yt[1] + what[2] * yt[2];
    *d = (u - pstar[0]) * (u - pstar[0]) + (v - pstar[1]) * (v - pstar[1]);
    *A = exp(-*d / delta);
    if (amb) {
        amb[0] = 0.0;
        if (e >= 0 && eps > 0) {
            /* a candidate is a tie if moving p' by eps could make it the closer one:
             * |d_c - d_e| <= 2 eps |q_c - q_e| (first order), plus 1e-6 relative for rounding */
            const double *we = cand + 3 * e;
            double qex = we[0] * xk[0] + we[1] * xk[1] + we[2] * xk[2];
            double qey = we[0] * yk[0] + we[1] * yk[1] + we[2] * yk[2];
            for (int c = 0; c < 3; ++c) {
                if (c == e) continue;
                const double *wq = cand + 3 * c;
                double qcx = wq[0] * xk[0] + wq[1] * xk[1] + wq[2] * xk[2];
                double qcy = wq[0] * yk[0] + wq[1] * yk[1] + wq[2] * yk[2];
                double sep = hypot(qcx - qex, qcy - qey);
                if (!(fabs(cd[c] - dX) <= 2.0 * eps * sep + 1e-6 * fmax(cd[c], dX))) continue;
                const double *wc = cand + 3 * c;
                double qx = wc[0] * xt[0] + wc[1] * xt[1] + wc[2] * xt[2];
                double qy = wc[0] * yt[0] + wc[1] * yt[1] + wc[2] * yt[2];
                double d2 = (u - qx) * (u - qx) + (v - qy) * (v - qy);
                double dA = fabs(exp(-d2 / delta) - *A);
                if (dA > amb[0]) amb[0] = dA;
            }
        }
    }
    return 1;
}

/* --------------------------------------------------------------- per-image state */

typedef struct {
    int N, S, k0, k1;
    int *sk;
    double *tk;
    double *key;          /* (S+1)*V*3 */
    unsigned char *valid; /* (S+1)*V */
    double *Q;            /* (S+1)*V*3 view coordinates */
    int behind;
} img_state;

static int img_init(const om_scene *sc, int b, img_state *st)
{
    memset(st, 0, sizeof(*st));
    st->N = sc->n_sub[b];
    st->S = om_segments(sc, b);
    st->k0 = sc->sub_range ? sc->sub_range[2 * b] : 0;
    st->k1 = sc->sub_range ? sc->sub_range[2 * b + 1] : st->N;
    st->sk = (int *)malloc(sizeof(int) * (size_t)st->N);
    st->tk = (double *)malloc(sizeof(double) * (size_t)st->N);
    if (om_schedule(st->N, st->S, sc->rule[b], st->sk, st->tk)) return -1;
    size_t nk = (size_t)(st->S + 1) * sc->V;
    st->key = (double *)malloc(sizeof(double) * 3 * nk);
    st->Q = (double *)malloc(sizeof(double) * 3 * nk);
    st->valid = (unsigned char *)malloc(nk);
    st->behind = om_keyframes(sc, b, st->key, st->valid, st->Q);
    return 0;
}

static void img_free(img_state *st)
{
    free(st->sk); free(st->tk); free(st->key); free(st->Q); free(st->valid);
}

/* Sub-frame geometry: screen-space lerp of keyframes s, s+1 at tau (Eq.5-6). */
static void lerp_subframe(const om_scene *sc, const img_state *st, int k, double *X, double *Y, double *Z,
                          unsigned char *ok)
{
    int s = st->sk[k];
    double tau = st->tk[k];
    const double *K0 = st->key + (size_t)3 * s * sc->V, *K1 = st->key + (size_t)3 * (s + 1) * sc->V;
    const unsigned char *v0 = st->valid + (size_t)s * sc->V, *v1 = st->valid + (size_t)(s + 1) * sc->V;
    for (int v = 0; v < sc->V; ++v) {
        X[v] = (1.0 - tau) * K0[3 * v] + tau * K1[3 * v];
        Y[v] = (1.0 - tau) * K0[3 * v + 1] + tau * K1[3 * v + 1];
        Z[v] = (1.0 - tau) * K0[3 * v + 2] + tau * K1[3 * v + 2];
        ok[v] = v0[v] && v1[v];
    }
}

static double pix_u(int i, int W) { return -1.0 + (2.0 * i + 1.0) / W; }   /* Q9 */
static double pix_v(int j, int H) { return 1.0 - (2.0 * j + 1.0) / H; }    /* Q9: row 0 at the top */

/* per-pixel candidate bookkeeping for the nominal z-buffer and the Q16 perturbed sets */
typedef struct {
    double z[3];      /* 0 nominal, 1 loose (-eps), 2 strict (+eps) */
    int id[3];
    double w[3];      /* nominal winner weights */
    double delta;     /* max |value change| of this sub-frame under the Q16 perturbations */
    int amb_id;       /* the winner (id) can change under the Q16 perturbations */
    double P;         /* soft background: prod_j (1 - A_j) (Eq.15) over all faces, uncovered pixels */
    double Pnz;       /*   the same product over the factors that are not exactly 0 */
    int nz;           /*   number of factors exactly 0 */
    int amb_soft;     /*   a closest-edge choice was a rounding-level tie (Q20) */
} pixstate;

static void ps_reset(pixstate *p)
{
    for (int i = 0; i < 3; ++i) { p->z[i] = INFINITY; p->id[i] = -1; }
    p->w[0] = p->w[1] = p->w[2] = 0;
    p->delta = 0;
    p->amb_id = 0;
    p->P = 1.0;
    p->Pnz = 1.0;
    p->nz = 0;
    p->amb_soft = 0;
}

typedef struct {
    double x[3], y[3], z[3];
    double len[3];     /* length of the edge opposite vertex i */
    double pad;        /* bbox padding for the loose set */
    int ok;
} face_geo;

static int face_setup(const om_scene *sc, int f, const double *X, const double *Y, const double *Z,
                      const unsigned char *okv, double eps, face_geo *g)
{
    const int *fv = sc->faces + 3 * f;
    g->ok = 0;
    for (int i = 0; i < 3; ++i)
        if (fv[i] < 0 || fv[i] >= sc->V || !okv[fv[i]]) return 0;
    for (int i = 0; i < 3; ++i) { g->x[i] = X[fv[i]]; g->y[i] = Y[fv[i]]; g->z[i] = Z[fv[i]]; }
    double det = g->x[0] * (g->y[1] - g->y[2]) - g->x[1] * (g->y[0] - g->y[2]) + g->x[2] * (g->y[0] - g->y[1]);
    if (!(fabs(det) > EPS_D)) return 0;
    g->pad = 1e-9;
    if (eps > 0) {
        double minsin = 1.0;
        for (int i = 0; i < 3; ++i) {
            int j = (i + 1) % 3, l = (i + 2) % 3;
            g->len[i] = hypot(g->x[l] - g->x[j], g->y[l] - g->y[j]);
        }
        for (int i = 0; i < 3; ++i) {   /* sin of the interior angle at vertex i */
            int j = (i + 1) % 3, l = (i + 2) % 3;
            double sn = fabs(det) / (g->len[j] * g->len[l]);
            if (sn < minsin) minsin = sn;
        }
        g->pad = 2.0 * eps / fmax(minsin * 0.5, 1e-12) + 1e-9;
        if (g->pad > 4.0) g->pad = 4.0;
    }
    g->ok = 1;
    return 1;
}

static void face_bbox(const face_geo *g, int H, int W, int *i0, int *i1, int *j0, int *j1)
{
    double xmn = fmin(g->x[0], fmin(g->x[1], g->x[2])) - g->pad;
    double xmx = fmax(g->x[0], fmax(g->x[1], g->x[2])) + g->pad;
    double ymn = fmin(g->y[0], fmin(g->y[1], g->y[2])) - g->pad;
    double ymx = fmax(g->y[0], fmax(g->y[1], g->y[2])) + g->pad;
    double a = ceil(((xmn + 1.0) * W - 1.0) * 0.5), bb = floor(((xmx + 1.0) * W - 1.0) * 0.5);
    double c = ceil(((1.0 - ymx) * H - 1.0) * 0.5), d = floor(((1.0 - ymn) * H - 1.0) * 0.5);
    *i0 = a < 0 ? 0 : (a > W ? W : (int)a);
    *i1 = bb > W - 1 ? W - 1 : (bb < -1 ? -1 : (int)bb);
    *j0 = c < 0 ? 0 : (c > H ? H : (int)c);
    *j1 = d > H - 1 ? H - 1 : (d < -1 ? -1 : (int)d);
}

typedef struct {
    double maxdev;      /* fast-solver vs textbook max |dw| over covered pairs with |D| > 1e-10 */
    double nchecked;
    double necessary;   /* covered (pixel, face, sub-frame) pairs */
    double covered;     /* covered (pixel, sub-frame) */
} om_stats_t;

/* per-sub-frame context for the ambiguity analysis */
typedef struct {
    const double *X, *Y, *Z;
    const unsigned char *okv;
    const int *nbr;    /* 3F: neighbour across the edge opposite corner i, as 3*g + i_g, or -1 */
} sub_ctx;

static int cmp_edge(const void *pa, const void *pb)
{
    const int *a = (const int *)pa, *b = (const int *)pb;
    if (a[0] != b[0]) return a[0] < b[0] ? -1 : 1;
    if (a[1] != b[1]) return a[1] < b[1] ? -1 : 1;
    return a[2] < b[2] ? -1 : (a[2] > b[2]);
}

/* Edge adjacency by vertex indices: two faces share an edge iff they share its two vertex
 * indices (edges with more than two faces are treated as boundaries). */
static int *build_nbr(const om_scene *sc)
{
    int F = sc->F;
    int *e = (int *)malloc(sizeof(int) * 3 * 3 * (size_t)(F > 0 ? F : 1));
    int *nbr = (int *)malloc(sizeof(int) * 3 * (size_t)(F > 0 ? F : 1));
    for (int f = 0; f < F; ++f)
        for (int i = 0; i < 3; ++i) {
            int a = sc->faces[3 * f + (i + 1) % 3], b = sc->faces[3 * f + (i + 2) % 3];
            int *r = e + 3 * (3 * f + i);
            r[0] = a < b ? a : b;
            r[1] = a < b ? b : a;
            r[2] = 3 * f + i;
            nbr[3 * f + i] = -1;
        }
    qsort(e, 3 * (size_t)F, 3 * sizeof(int), cmp_edge);
    for (int q = 0; q < 3 * F;) {
        int r = q + 1;
        while (r < 3 * F && e[3 * r] == e[3 * q] && e[3 * r + 1] == e[3 * q + 1]) ++r;
        if (r - q == 2) {
            nbr[e[3 * q + 2]] = e[3 * (q + 1) + 2];
            nbr[e[3 * (q + 1) + 2]] = e[3 * q + 2];
        }
        q = r;
    }
    free(e);
    return nbr;
}

/* Q16 strict scenario (inside test at +eps), watertight reading: a nominally covering face whose
 * pixel lies within eps of one of its edges is dropped, unless across every such edge the
 * neighbouring face (same two vertex indices) lies on the other side of the edge at this pixel --
 * then the pixel belongs to one of the two faces under any consistent rounding (no crack can open
 * inside a mesh), which the loose scenario and the depth ties already cover. */
static int strict_member(const om_scene *sc, const sub_ctx *cx, int f, const double w[3], double ad,
                         const double len[3], double u, double v, double eps)
{
    for (int i = 0; i < 3; ++i) {
        double sd = w[i] * ad / len[i];
        if (sd >= eps) continue;
        int nb = cx->nbr[3 * f + i];
        if (nb < 0) return 0;
        int g = nb / 3, ig = nb % 3;
        face_geo gg;
        if (!face_setup(sc, g, cx->X, cx->Y, cx->Z, cx->okv, eps, &gg)) return 0;
        double wg[3], detg;
        if (!om_bary_textbook(gg.x, gg.y, u, v, wg, &detg)) return 0;
        double sdg = wg[ig] * fabs(detg) / gg.len[ig];
        if (!(sdg <= 0.0)) return 0;      /* same side (a fold) or no neighbour coverage */
    }
    return 1;
}

/* pass 1 per pair: nominal / loose / strict z-buffers */
static void pair_pass1(const om_scene *sc, const sub_ctx *cx, const face_geo *g, int f, double u, double v,
                       double eps, pixstate *ps, const img_state *st, int k, om_stats_t *stt, int check_fast)
{
    double w[3], det;
    if (!om_bary_textbook(g->x, g->y, u, v, w, &det)) return;
    double z = w[0] * g->z[0] + w[1] * g->z[1] + w[2] * g->z[2];
    int cov = (w[0] >= 0.0) && (w[1] >= 0.0) && (w[2] >= 0.0);
    if (cov) {
        if (stt) stt->necessary += 1;
        if (z < ps->z[0]) {
            ps->z[0] = z; ps->id[0] = f;
            ps->w[0] = w[0]; ps->w[1] = w[1]; ps->w[2] = w[2];
        }
        if (check_fast && stt) {
            const int *fv = sc->faces + 3 * f;
            int s = st->sk[k];
            double X0[3], Y0[3], X1[3], Y1[3], wf[3], den;
            for (int i = 0; i < 3; ++i) {
                X0[i] = st->key[3 * ((size_t)s * sc->V + fv[i])];
                Y0[i] = st->key[3 * ((size_t)s * sc->V + fv[i]) + 1];
                X1[i] = st->key[3 * ((size_t)(s + 1) * sc->V + fv[i])];
                Y1[i] = st->key[3 * ((size_t)(s + 1) * sc->V + fv[i]) + 1];
            }
            if (om_fast_eval(X0, Y0, X1, Y1, u, v, st->tk[k], wf, &den) && fabs(den) > 1e-10) {
                for (int i = 0; i < 3; ++i) {
                    double d = fabs(wf[i] - w[i]);
                    if (d > stt->maxdev) stt->maxdev = d;
                }
                stt->nchecked += 1;
            }
        }
    }
    if (eps > 0) {
        double ad = fabs(det), sdmin = INFINITY;
        for (int i = 0; i < 3; ++i) {
            double sd = w[i] * ad / g->len[i];
            if (sd < sdmin) sdmin = sd;
        }
        if (sdmin >= -eps && z < ps->z[1]) { ps->z[1] = z; ps->id[1] = f; }
        if (cov && z < ps->z[2] && (sdmin >= eps || strict_member(sc, cx, f, w, ad, g->len, u, v, eps))) {
            ps->z[2] = z;
            ps->id[2] = f;
        }
    }
}

static void shade_w(const om_scene *sc, int f, const double w[3], double rgb[3])
{
    const int *fv = sc->faces + 3 * f;
    for (int c = 0; c < 3; ++c)
        rgb[c] = w[0] * sc->colors[3 * fv[0] + c] + w[1] * sc->colors[3 * fv[1] + c] + w[2] * sc->colors[3 * fv[2] + c];
}

/* pass 2 per pair (ambiguity): any face within the depth tolerance of a set's minimum is a
 * possible outcome (Q16); record how far its shaded value is from the nominal one and whether its
 * id differs. */
static void pair_pass2(const om_scene *sc, const sub_ctx *cx, const face_geo *g, int f, double u, double v,
                       double eps, const om_opts *op, pixstate *ps, const double nom_rgb[3])
{
    double w[3], det;
    if (!om_bary_textbook(g->x, g->y, u, v, w, &det)) return;
    double z = w[0] * g->z[0] + w[1] * g->z[1] + w[2] * g->z[2];
    double ad = fabs(det), sdmin = INFINITY;
    for (int i = 0; i < 3; ++i) {
        double sd = w[i] * ad / g->len[i];
        if (sd < sdmin) sdmin = sd;
    }
    const int cov = w[0] >= 0 && w[1] >= 0 && w[2] >= 0;
    int in[3] = {cov, sdmin >= -eps,
                 cov && (sdmin >= eps || strict_member(sc, cx, f, w, ad, g->len, u, v, eps))};
    for (int sidx = 0; sidx < 3; ++sidx) {
        if (!in[sidx] || !(ps->z[sidx] < INFINITY)) continue;
        if (z <= ps->z[sidx] + op->amb_z_rel * fabs(ps->z[sidx])) {
            if (f != ps->id[0]) ps->amb_id = 1;
            double rgb[3];
            shade_w(sc, f, w, rgb);
            if (ps->id[0] < 0) {
                ps->delta = fmax(ps->delta, 1.0);
            } else {
                for (int c = 0; c < 3; ++c) ps->delta = fmax(ps->delta, fabs(rgb[c] - nom_rgb[c]));
            }
        }
    }
}

static void pix_finalize_amb(pixstate *ps)
{
    /* a perturbed set that is empty while the nominal pixel is covered (or vice versa):
     * the alpha channel changes by 1 */
    for (int sidx = 1; sidx < 3; ++sidx) {
        if ((ps->id[sidx] < 0) != (ps->id[0] < 0)) { ps->delta = fmax(ps->delta, 1.0); ps->amb_id = 1; }
    }
}

/* Keyframe triangles of face f in segment s (NDC x, y of keyframes s and s+1). */
static void face_keys(const om_scene *sc, const img_state *st, int s, int f, double X0[3], double Y0[3],
                      double X1[3], double Y1[3])
{
    const int *fv = sc->faces + 3 * f;
    for (int i = 0; i < 3; ++i) {
        const double *a = st->key + 3 * ((size_t)s * sc->V + fv[i]);
        const double *b = st->key + 3 * ((size_t)(s + 1) * sc->V + fv[i]);
        X0[i] = a[0]; Y0[i] = a[1];
        X1[i] = b[0]; Y1[i] = b[1];
    }
}

/* Fold one face's background term into an uncovered pixel's product (Eq.15). */
static void soft_accum(pixstate *ps, double A, double ambA)
{
    double fac = 1.0 - A;
    ps->P *= fac;
    if (fac == 0.0) ps->nz += 1;
    else ps->Pnz *= fac;
    if (ambA > 0.0) ps->delta += ambA;          /* value-change bound: d alpha / d A_j <= 1 */
    if (ambA > 1e-6) ps->amb_soft = 1;          /* gradient comparison: a tie that moves A by > 1e-6 (Q20) */
}

/* Pixel range whose soft term can be non-zero: the box of F(tau) grown by sqrt(760 delta) (beyond
 * it d / delta > 760 and exp(-d / delta) is exactly 0 in fp64, so skipping those factors of exactly
 * 1 leaves the product bit-identical to the brute loop).  Returns 0 if empty. */
static int soft_range(const face_geo *g, double delta, int H, int W, int *i0, int *i1, int *j0, int *j1)
{
    face_geo gg = *g;
    gg.pad = sqrt(760.0 * delta) + 1e-9;
    face_bbox(&gg, H, W, i0, i1, j0, j1);
    return *i0 <= *i1 && *j0 <= *j1;
}

/* Soft background pass of one sub-frame: for every nominally uncovered pixel, the product over all
 * faces valid at tau, in face-index order. */
static void soft_subframe(const om_scene *sc, const om_opts *op, const img_state *st, int k, pixstate *ps,
                          const int *pix_idx, int npix, const double *X, const double *Y, const double *Z,
                          const unsigned char *okv)
{
    int H = sc->H, W = sc->W;
    int s = st->sk[k];
    double tau = st->tk[k];
    face_geo g;
    double X0[3], Y0[3], X1[3], Y1[3], A, d, wh[3], ps2[2], amb;
    if (pix_idx) {
        for (int q = 0; q < npix; ++q) {
            if (ps[q].id[0] >= 0) continue;
            int p = pix_idx[q];
            double u = pix_u(p % W, W), v = pix_v(p / W, H);
            for (int f = 0; f < sc->F; ++f) {
                if (!face_setup(sc, f, X, Y, Z, okv, 0.0, &g)) continue;
                face_keys(sc, st, s, f, X0, Y0, X1, Y1);
                if (!om_soft_pair(X0, Y0, X1, Y1, tau, u, v, op->delta, op->soft_exact, op->eps_amb, &A, &d, wh, ps2,
                                  &amb))
                    continue;
                soft_accum(&ps[q], A, amb);
            }
        }
        return;
    }
    for (int f = 0; f < sc->F; ++f) {
        if (!face_setup(sc, f, X, Y, Z, okv, 0.0, &g)) continue;
        int i0 = 0, i1 = W - 1, j0 = 0, j1 = H - 1;
        if (op->mode == 1 && !soft_range(&g, op->delta, H, W, &i0, &i1, &j0, &j1)) continue;
        face_keys(sc, st, s, f, X0, Y0, X1, Y1);
        for (int j = j0; j <= j1; ++j)
            for (int i = i0; i <= i1; ++i) {
                pixstate *pp = &ps[j * W + i];
                if (pp->id[0] >= 0) continue;
                if (!om_soft_pair(X0, Y0, X1, Y1, tau, pix_u(i, W), pix_v(j, H), op->delta, op->soft_exact, op->eps_amb,
                                  &A, &d, wh, ps2, &amb))
                    continue;
                soft_accum(pp, A, amb);
            }
    }
}

/* Render one sub-frame (b, k) into per-pixel states.  pix_idx == NULL: all pixels (brute or
 * binned); otherwise only the listed pixel indices (brute over faces). */
static void render_subframe(const om_scene *sc, const om_opts *op, const img_state *st, int k,
                            pixstate *ps, const int *pix_idx, int npix, om_stats_t *stt,
                            double *X, double *Y, double *Z, unsigned char *okv, const int *nbr)
{
    int H = sc->H, W = sc->W, P = H * W;
    double eps = op->eps_amb;
    lerp_subframe(sc, st, k, X, Y, Z, okv);
    sub_ctx cxv = {X, Y, Z, okv, nbr};
    const sub_ctx *cx = &cxv;
    int nloop = pix_idx ? npix : P;
    for (int q = 0; q < nloop; ++q) ps_reset(&ps[q]);
    face_geo g;
    if (pix_idx) {
        for (int q = 0; q < npix; ++q) {
            int p = pix_idx[q], i = p % W, j = p / W;
            double u = pix_u(i, W), v = pix_v(j, H);
            for (int f = 0; f < sc->F; ++f) {
                if (!face_setup(sc, f, X, Y, Z, okv, eps, &g)) continue;
                pair_pass1(sc, cx, &g, f, u, v, eps, &ps[q], st, k, stt, op->check_fast);
            }
            if (eps > 0) {
                double nom[3] = {0, 0, 0};
                if (ps[q].id[0] >= 0) shade_w(sc, ps[q].id[0], ps[q].w, nom);
                for (int f = 0; f < sc->F; ++f) {
                    if (!face_setup(sc, f, X, Y, Z, okv, eps, &g)) continue;
                    pair_pass2(sc, cx, &g, f, u, v, eps, op, &ps[q], nom);
                }
                pix_finalize_amb(&ps[q]);
            }
        }
        if (op->delta > 0) soft_subframe(sc, op, st, k, ps, pix_idx, npix, X, Y, Z, okv);
        return;
    }
    for (int f = 0; f < sc->F; ++f) {
        if (!face_setup(sc, f, X, Y, Z, okv, eps, &g)) continue;
        int i0 = 0, i1 = W - 1, j0 = 0, j1 = H - 1;
        if (op->mode == 1) face_bbox(&g, H, W, &i0, &i1, &j0, &j1);
        for (int j = j0; j <= j1; ++j)
            for (int i = i0; i <= i1; ++i)
                pair_pass1(sc, cx, &g, f, pix_u(i, W), pix_v(j, H), eps, &ps[j * W + i], st, k, stt, op->check_fast);
    }
    if (eps > 0) {
        double *nom = (double *)malloc(sizeof(double) * 3 * (size_t)P);
        for (int p = 0; p < P; ++p) {
            nom[3 * p] = nom[3 * p + 1] = nom[3 * p + 2] = 0;
            if (ps[p].id[0] >= 0) shade_w(sc, ps[p].id[0], ps[p].w, nom + 3 * p);
        }
        for (int f = 0; f < sc->F; ++f) {
            if (!face_setup(sc, f, X, Y, Z, okv, eps, &g)) continue;
            int i0 = 0, i1 = W - 1, j0 = 0, j1 = H - 1;
            if (op->mode == 1) face_bbox(&g, H, W, &i0, &i1, &j0, &j1);
            for (int j = j0; j <= j1; ++j)
                for (int i = i0; i <= i1; ++i)
                    pair_pass2(sc, cx, &g, f, pix_u(i, W), pix_v(j, H), eps, op, &ps[j * W + i], nom + 3 * (j * W + i));
        }
        for (int p = 0; p < P; ++p) pix_finalize_amb(&ps[p]);
        free(nom);
    }
    if (op->delta > 0) soft_subframe(sc, op, st, k, ps, NULL, P, X, Y, Z, okv);
}

static int nthreads_of(const om_opts *op)
{
#ifdef _OPENMP
    return op->threads > 0 ? op->threads : omp_get_max_threads();
#else
    (void)op;
    return 1;
#endif
}

/* list of pixel indices of image b in pixel-list mode; returns count, fills idx and map to list slot */
static int pixlist_for(const om_opts *op, int b, int W, int *idx, int *slot)
{
    int n = 0;
    for (int q = 0; q < op->npix; ++q)
        if (op->pix[3 * q] == b) { idx[n] = op->pix[3 * q + 1] * W + op->pix[3 * q + 2]; slot[n] = q; ++n; }
    return n;
}

/* Forward render.
 *   out_rgba: B*H*W*4 (full mode) or npix*4 (pixel-list mode): (1/N) * sum over k in [k0,k1)
 *   ids: B*H*W (or npix) winner id at sub-frame ids_k (-1 none), may be NULL
 *   amb_img / amb_ids / amb_win: Q16 ambiguity flags (need eps_amb > 0), may be NULL:
 *     amb_img: the Q16 perturbations can move the BLURRED value by more than amb_val_tol
 *              (sum over sub-frames of the per-sub-frame change / N);
 *     amb_ids: the winner at sub-frame ids_k can change;
 *     amb_win: the winner can change at some sub-frame (gradient exclusion, Q18)
 *   frozen: per (b, k, pixel) face ids [sum_b N_b * H * W]; when non-NULL the value of each
 *           (pixel, k) is evaluated for the given face without a coverage test (frozen-visibility
 *           forward used by the finite-difference pin; full mode only)
 *   stats: om_stats_t (4 doubles) or NULL
 * Returns 0 ok, 1 a vertex was behind the near plane (its faces skipped), -1 invalid input. */
int om_render_fwd(const om_scene *sc, const om_opts *op, double *out_rgba, int *ids, int ids_k,
                  unsigned char *amb_img, unsigned char *amb_ids, unsigned char *amb_win, const int *frozen,
                  double *stats)
{
    int H = sc->H, W = sc->W, P = H * W, ret = 0;
    int list = op->npix > 0;
    int nout = list ? op->npix : sc->B * P;
    memset(out_rgba, 0, sizeof(double) * 4 * (size_t)nout);
    if (ids) for (int q = 0; q < nout; ++q) ids[q] = -1;
    if (amb_img) memset(amb_img, 0, (size_t)nout);
    if (amb_ids) memset(amb_ids, 0, (size_t)nout);
    if (amb_win) memset(amb_win, 0, (size_t)nout);
    om_stats_t tot = {0, 0, 0, 0};
    size_t frozen_off = 0;
    int *nbr = op->eps_amb > 0 ? build_nbr(sc) : NULL;
    int *lidx = (int *)malloc(sizeof(int) * (size_t)(op->npix + 1));
    int *lslot = (int *)malloc(sizeof(int) * (size_t)(op->npix + 1));
    for (int b = 0; b < sc->B; ++b) {
        img_state st;
        if (img_init(sc, b, &st)) { img_free(&st); ret = -1; break; }
        if (st.behind) ret = 1;
        int np = list ? pixlist_for(op, b, W, lidx, lslot) : P;
        int nth = nthreads_of(op);
        if (nth > st.N) nth = st.N;
        if (nth < 1) nth = 1;
        double *acc = (double *)calloc((size_t)nth * 5 * np, sizeof(double));   /* rgba + sum delta/N */
        om_stats_t *tst = (om_stats_t *)calloc((size_t)nth, sizeof(om_stats_t));
        int N = st.N;
#pragma omp parallel num_threads(nth)
        {
            int tid = 0;
#ifdef _OPENMP
            tid = omp_get_thread_num();
#endif
            pixstate *ps = (pixstate *)malloc(sizeof(pixstate) * (size_t)(np > 0 ? np : 1));
            double *X = (double *)malloc(sizeof(double) * (size_t)(sc->V + 1));
            double *Y = (double *)malloc(sizeof(double) * (size_t)(sc->V + 1));
            double *Z = (double *)malloc(sizeof(double) * (size_t)(sc->V + 1));
            unsigned char *okv = (unsigned char *)malloc((size_t)(sc->V + 1));
            double *a = acc + (size_t)tid * 5 * np;
#pragma omp for schedule(static)
            for (int k = st.k0; k < st.k1; ++k) {
                if (frozen) {
                    /* frozen-visibility evaluation (FD pin only) */
                    lerp_subframe(sc, &st, k, X, Y, Z, okv);
                    const int *fz = frozen + frozen_off + (size_t)k * P;
                    if (op->delta > 0) {   /* frozen coverage: soft alpha of the frozen-uncovered pixels */
                        for (int p = 0; p < P; ++p) { ps_reset(&ps[p]); ps[p].id[0] = fz[p]; }
                        soft_subframe(sc, op, &st, k, ps, NULL, P, X, Y, Z, okv);
                        for (int p = 0; p < P; ++p)
                            if (fz[p] < 0) a[5 * p + 3] += 1.0 - ps[p].P;
                    }
                    for (int p = 0; p < P; ++p) {
                        int f = fz[p];
                        if (f < 0) continue;
                        face_geo g;
                        if (!face_setup(sc, f, X, Y, Z, okv, 0.0, &g)) continue;
                        double w[3], det, rgb[3];
                        if (!om_bary_textbook(g.x, g.y, pix_u(p % W, W), pix_v(p / W, H), w, &det)) continue;
                        shade_w(sc, f, w, rgb);
                        a[5 * p] += rgb[0]; a[5 * p + 1] += rgb[1]; a[5 * p + 2] += rgb[2]; a[5 * p + 3] += 1.0;
                    }
                    continue;
                }
                render_subframe(sc, op, &st, k, ps, list ? lidx : NULL, np, &tst[tid], X, Y, Z, okv, nbr);
                for (int q = 0; q < np; ++q) {
                    int oq = list ? lslot[q] : b * P + q;
                    if (ps[q].id[0] >= 0) {
                        double rgb[3];
                        shade_w(sc, ps[q].id[0], ps[q].w, rgb);      /* Eq.9 */
                        a[5 * q] += rgb[0]; a[5 * q + 1] += rgb[1]; a[5 * q + 2] += rgb[2]; a[5 * q + 3] += 1.0;
                        tst[tid].covered += 1;
                    } else if (op->delta > 0) {
                        a[5 * q + 3] += 1.0 - ps[q].P;                 /* A_i(t), Eq.15 (background RGB 0) */
                    }
                    a[5 * q + 4] += ps[q].delta;
                    if (ids && k == ids_k) ids[oq] = ps[q].id[0];
                    if (amb_win && (ps[q].amb_id || ps[q].amb_soft)) amb_win[oq] = 1;    /* distinct k write the same 1 */
                    if (amb_ids && k == ids_k && ps[q].amb_id) amb_ids[oq] = 1;
                }
            }
            free(ps); free(X); free(Y); free(Z); free(okv);
        }
        for (int q = 0; q < np; ++q) {
            int oq = list ? lslot[q] : b * P + q;
            for (int c = 0; c < 4; ++c) {
                double s = 0;
                for (int t = 0; t < nth; ++t) s += acc[(size_t)t * 5 * np + 5 * q + c];
                out_rgba[4 * (size_t)oq + c] = s / (double)N;   /* uniform mean */
            }
            if (amb_img) {
                double d = 0;
                for (int t = 0; t < nth; ++t) d += acc[(size_t)t * 5 * np + 5 * q + 4];
                if (d / (double)N > op->amb_val_tol) amb_img[oq] = 1;
            }
        }
        for (int t = 0; t < nth; ++t) {
            if (tst[t].maxdev > tot.maxdev) tot.maxdev = tst[t].maxdev;
            tot.nchecked += tst[t].nchecked;
            tot.necessary += tst[t].necessary;
            tot.covered += tst[t].covered;
        }
        free(acc); free(tst);
        frozen_off += (size_t)N * P;
        img_free(&st);
    }
    free(lidx); free(lslot); free(nbr);
    if (stats) { stats[0] = tot.maxdev; stats[1] = tot.nchecked; stats[2] = tot.necessary; stats[3] = tot.covered; }
    return ret;
}

/* Soft background gradient of one sub-frame (P:L341-342 through Eq.10-15; w^* frozen; Q11):
 * for an uncovered pixel with alpha = 1 - prod_j (1 - A_j) and G_a = dL/dalpha_k,
 *   dalpha/dA_j = prod_{l != j} (1 - A_l)  (Pnz / (1 - A_j) when no factor is 0; Pnz for the single
 *                 zero factor; 0 otherwise),  dA_j/dd = -A_j / delta,
 *   dd/dv_i(tau) = -2 w^*_i (p - F(tau) w^*)  (Eq.14 with w^* constant),
 * then split (1 - tau), tau onto the keyframes like the foreground term. */
static void soft_grad_subframe(const om_scene *sc, const om_opts *op, const img_state *st, int k,
                               const pixstate *ps, const int *pix_idx, int npix, const double *gal,
                               const double *X, const double *Y, const double *Z, const unsigned char *okv,
                               double *mk)
{
    int H = sc->H, W = sc->W, V = sc->V;
    int s = st->sk[k];
    double tau = st->tk[k];
    face_geo g;
    double X0[3], Y0[3], X1[3], Y1[3], A, d, wh[3], pst[2];
    for (int f = 0; f < sc->F; ++f) {
        if (!face_setup(sc, f, X, Y, Z, okv, 0.0, &g)) continue;
        int i0 = 0, i1 = W - 1, j0 = 0, j1 = H - 1;
        if (!pix_idx && op->mode == 1 && !soft_range(&g, op->delta, H, W, &i0, &i1, &j0, &j1)) continue;
        face_keys(sc, st, s, f, X0, Y0, X1, Y1);
        const int *fv = sc->faces + 3 * f;
        int bw = i1 - i0 + 1, nloop = pix_idx ? npix : bw * (j1 - j0 + 1);
        for (int r = 0; r < nloop; ++r) {
            int q = pix_idx ? r : (j0 + r / bw) * W + i0 + r % bw;
            int p = pix_idx ? pix_idx[r] : q;
            int i = p % W, j = p / W;
            const pixstate *pp = &ps[q];
            if (pp->id[0] >= 0 || gal[q] == 0.0) continue;
            double u = pix_u(i, W), v = pix_v(j, H);
            if (!om_soft_pair(X0, Y0, X1, Y1, tau, u, v, op->delta, op->soft_exact, 0.0, &A, &d, wh, pst, NULL)) continue;
            if (A == 0.0) continue;
            double fac = 1.0 - A, dadA;
            if (pp->nz == 0) dadA = pp->Pnz / fac;
            else if (pp->nz == 1 && fac == 0.0) dadA = pp->Pnz;
            else dadA = 0.0;
            double c = gal[q] * dadA * A / op->delta * 2.0;
            for (int a = 0; a < 3; ++a) {
                if (wh[a] == 0.0) continue;
                double gx = c * wh[a] * (u - pst[0]), gy = c * wh[a] * (v - pst[1]);
                size_t o0 = ((size_t)s * V + fv[a]) * 2, o1 = ((size_t)(s + 1) * V + fv[a]) * 2;
                mk[o0] += (1.0 - tau) * gx; mk[o0 + 1] += (1.0 - tau) * gy;
                mk[o1] += tau * gx;         mk[o1 + 1] += tau * gy;
            }
        }
    }
}

/* Backward (frozen winners Q11).
 *   grad_rgba: dL/dI, B*H*W*4 (or npix*4 in pixel-list mode; the gradient is then the one of a
 *              loss that only reads the listed pixels)
 *   dverts, dcolors: V*3 outputs (overwritten)
 *   dkey: optional sum_b (S_b+1)*V*2 screen-space keyframe gradients (overwritten)
 * Alpha carries no position gradient in the hard-coverage path; with op->delta > 0 the
 * background alpha of Eq.10-15 does (soft_grad_subframe). */
int om_render_bwd(const om_scene *sc, const om_opts *op, const double *grad_rgba, double *dverts,
                  double *dcolors, double *dkey)
{
    int H = sc->H, W = sc->W, P = H * W, V = sc->V, ret = 0;
    int list = op->npix > 0;
    memset(dverts, 0, sizeof(double) * 3 * (size_t)V);
    memset(dcolors, 0, sizeof(double) * 3 * (size_t)V);
    size_t dkey_off = 0;
    int *lidx = (int *)malloc(sizeof(int) * (size_t)(op->npix + 1));
    int *lslot = (int *)malloc(sizeof(int) * (size_t)(op->npix + 1));
    om_opts op1 = *op;
    op1.eps_amb = 0;          /* ambiguity analysis is a forward-only diagnostic */
    op1.check_fast = 0;
    for (int b = 0; b < sc->B; ++b) {
        img_state st;
        if (img_init(sc, b, &st)) { img_free(&st); ret = -1; break; }
        if (st.behind) ret = 1;
        int S = st.S, N = st.N;
        int np = list ? pixlist_for(op, b, W, lidx, lslot) : P;
        int nth = nthreads_of(op);
        if (nth > N) nth = N;
        if (nth < 1) nth = 1;
        size_t nkv = (size_t)(S + 1) * V * 2;
        double *gk = (double *)calloc((size_t)nth * nkv, sizeof(double));
        double *gc = (double *)calloc((size_t)nth * 3 * V, sizeof(double));
#pragma omp parallel num_threads(nth)
        {
            int tid = 0;
#ifdef _OPENMP
            tid = omp_get_thread_num();
#endif
            pixstate *ps = (pixstate *)malloc(sizeof(pixstate) * (size_t)(np > 0 ? np : 1));
            double *X = (double *)malloc(sizeof(double) * (size_t)(V + 1));
            double *Y = (double *)malloc(sizeof(double) * (size_t)(V + 1));
            double *Z = (double *)malloc(sizeof(double) * (size_t)(V + 1));
            unsigned char *okv = (unsigned char *)malloc((size_t)(V + 1));
            double *mk = gk + (size_t)tid * nkv, *mc = gc + (size_t)tid * 3 * V;
            double *gal = op->delta > 0 ? (double *)malloc(sizeof(double) * (size_t)(np > 0 ? np : 1)) : NULL;
#pragma omp for schedule(static)
            for (int k = st.k0; k < st.k1; ++k) {
                render_subframe(sc, &op1, &st, k, ps, list ? lidx : NULL, np, NULL, X, Y, Z, okv, NULL);
                int s = st.sk[k];
                double tau = st.tk[k];
                if (gal) {   /* soft background: dL/dalpha_k = G_alpha / N */
                    for (int q = 0; q < np; ++q) gal[q] = grad_rgba[4 * (size_t)(list ? lslot[q] : b * P + q) + 3] / N;
                    soft_grad_subframe(sc, &op1, &st, k, ps, list ? lidx : NULL, np, gal, X, Y, Z, okv, mk);
                }
                for (int q = 0; q < np; ++q) {
                    int f = ps[q].id[0];
                    if (f < 0) continue;
                    const double *G = grad_rgba + 4 * (size_t)(list ? lslot[q] : b * P + q);
                    double g[3] = {G[0] / N, G[1] / N, G[2] / N};   /* d(mean over N)/dI_k */
                    const int *fv = sc->faces + 3 * f;
                    double x[3], y[3];
                    for (int i = 0; i < 3; ++i) { x[i] = X[fv[i]]; y[i] = Y[fv[i]]; }
                    double det = x[0] * (y[1] - y[2]) - x[1] * (y[0] - y[2]) + x[2] * (y[0] - y[1]);
                    const double *w = ps[q].w;
                    /* dI/dc_i = w_i (Eq.9) */
                    for (int i = 0; i < 3; ++i)
                        for (int c = 0; c < 3; ++c) mc[3 * fv[i] + c] += w[i] * g[c];
                    /* dw_j/dp = first two columns of adj(F)/det (A9 rows) */
                    double dwdu[3] = {(y[1] - y[2]) / det, (y[2] - y[0]) / det, (y[0] - y[1]) / det};
                    double dwdv[3] = {(x[2] - x[1]) / det, (x[0] - x[2]) / det, (x[1] - x[0]) / det};
                    double sj[3];
                    for (int j = 0; j < 3; ++j) {
                        const double *cj = sc->colors + 3 * fv[j];
                        sj[j] = g[0] * cj[0] + g[1] * cj[1] + g[2] * cj[2];
                    }
                    double su = sj[0] * dwdu[0] + sj[1] * dwdu[1] + sj[2] * dwdu[2];
                    double sv = sj[0] * dwdv[0] + sj[1] * dwdv[1] + sj[2] * dwdv[2];
                    for (int i = 0; i < 3; ++i) {
                        /* dL/dv_i(tau) = -w_i * (sum_j s_j dw_j/dp); v_i(tau) = (1-tau) v_i^s + tau v_i^{s+1} */
                        double gx = -w[i] * su, gy = -w[i] * sv;
                        size_t o0 = ((size_t)s * V + fv[i]) * 2, o1 = ((size_t)(s + 1) * V + fv[i]) * 2;
                        mk[o0] += (1.0 - tau) * gx; mk[o0 + 1] += (1.0 - tau) * gy;
                        mk[o1] += tau * gx;         mk[o1 + 1] += tau * gy;
                    }
                }
            }
            free(ps); free(X); free(Y); free(Z); free(okv); free(gal);
        }
        /* reduce thread partials (static order) */
        double *K = (double *)calloc(nkv, sizeof(double));
        for (int t = 0; t < nth; ++t) {
            for (size_t i = 0; i < nkv; ++i) K[i] += gk[(size_t)t * nkv + i];
            for (int i = 0; i < 3 * V; ++i) dcolors[i] += gc[(size_t)t * 3 * V + i];
        }
        if (dkey) memcpy(dkey + dkey_off, K, sizeof(double) * nkv);
        dkey_off += nkv;
        /* chain keyframe screen gradients to world vertices:
         * x = Qx/(Qz ta), y = Qy/(Qz ta) (A34); Q = Rc (P - E); P = R_s (P0 - c) + c + T_s. */
        double Rc[9];
        cam_frame(sc->cams + 11 * b, Rc);
        double ta = tan(sc->cams[11 * b + 9]);
        for (int s = 0; s <= S; ++s) {
            double R[9], tr[3];
            pose_rt(sc, b, (double)s / (double)S, R, tr);
            for (int v = 0; v < V; ++v) {
                size_t o = (size_t)s * V + v;
                double gx = K[2 * o], gy = K[2 * o + 1];
                if (gx == 0.0 && gy == 0.0) continue;
                const double *Q = st.Q + 3 * o;
                double iz = 1.0 / (Q[2] * ta);
                /* dL/dQ = J^T (gx, gy), J = [[1/(z ta), 0, -Qx/(z^2 ta)], [0, 1/(z ta), -Qy/(z^2 ta)]] */
                double dQ[3] = {gx * iz, gy * iz, -(gx * Q[0] + gy * Q[1]) * iz / Q[2]};
                double dP[3];   /* Rc^T dQ */
                for (int i = 0; i < 3; ++i) dP[i] = Rc[i] * dQ[0] + Rc[3 + i] * dQ[1] + Rc[6 + i] * dQ[2];
                for (int i = 0; i < 3; ++i)   /* R_s^T dP (identity for static / translation) */
                    dverts[3 * v + i] += R[i] * dP[0] + R[3 + i] * dP[1] + R[6 + i] * dP[2];
            }
        }
        free(K); free(gk); free(gc);
        img_free(&st);
    }
    free(lidx); free(lslot);
    return ret;
}

int om_num_threads(int req)
{
#ifdef _OPENMP
    return req > 0 ? req : omp_get_max_threads();
#else
    (void)req;
    return 1;
#endif
}
