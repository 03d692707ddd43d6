/*
 * blurrast_optim.h -- C ABI of the translational inverse-rendering step of arxiv 2602.07860
 * (NEXT-4; section 5.1, Eq.16-17, appendix "Details of Loss Terms" A21-A22, "Hyperparameter
 * Settings" P:L1467-1474).  Together with blur_render_fwd / blur_render_bwd (blurrast.h) these are
 * the kernels of one recovery iteration: render -> L1 image loss -> backward -> regularisers ->
 * Adam, all on the device.  Same conventions as blurrast.h: device pointers unless "host", work
 * enqueued on `stream`, argument errors returned synchronously (blur_last_error()), the caller owns
 * every buffer.  Losses are written to device floats (overwritten); gradient outputs named
 * "grad_verts (+=)" are ACCUMULATED into, so the image gradient of blur_render_bwd and the
 * weighted regulariser gradients sum in one buffer.  Summation order in the loss scalars and in
 * the scattered gradients uses atomics (not bitwise reproducible; the values are).
 */
#ifndef BLURRAST_OPTIM_H
#define BLURRAST_OPTIM_H

#include <stddef.h>
#include <stdint.h>

#include "blurrast.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Mesh topology for the regularisers, built once per mesh from host faces [F,3]:
 *   N(v) = vertices sharing an edge with v (CSR, sorted), and the edges shared by exactly two faces
 *   (a < b, opposite vertices c, d), plus a 3V-float scratch area used by the Laplacian.
 * blur_topology_bytes: device bytes needed (0 + blur_last_error() on invalid faces).
 * blur_topology_build: builds on the host and copies into `topo` (device, >= bytes); synchronises
 * `stream` before returning (the host staging buffer is freed). */
size_t blur_topology_bytes(int V, int F, const int32_t *faces_host);
int blur_topology_build(int V, int F, const int32_t *faces_host, void *topo, size_t topo_bytes,
                        blur_stream_t stream);

/* Image loss Eq.16: loss[0] = sum |out - target|_rgb / (3 n) + sum |out - target|_a / n
 * over the n = n_images * H * W pixels of the images with image_mask[b] != 0 (device uint8 [B], or
 * NULL = all B images and n_images = B); grad [B,H,W,4] OVERWRITTEN with sign(out - target) / (3n)
 * (rgb) and / n (alpha), 0 for masked-out images; sign(0) = 0 (mean reduction: reading Q22). */
int blur_l1_loss_grad(const float *out, const float *target, int B, int H, int W, const uint8_t *image_mask,
                      int n_images, float *loss, float *grad, blur_stream_t stream);

/* Laplacian loss A21: loss[0] = sum_v || delta_v - mean_{v' in N(v)} delta_v' ||^2,
 * delta = verts - verts0 ([V,3] each); grad_verts (+=) weight * dL/dverts.  Vertices without
 * neighbours contribute nothing.  topo: from blur_topology_build (its scratch is written). */
int blur_laplacian_loss_grad(const float *verts, const float *verts0, int V, void *topo, float weight,
                             float *loss, float *grad_verts, blur_stream_t stream);

/* Smoothness loss A22: loss[0] = sum over the interior edges of (cos theta + 1)^2,
 * theta the dihedral angle between the two faces (pi when flat): cos theta = u.w / (|u||w|) with u,
 * w the components of c - a and d - a perpendicular to the edge b - a.  grad_verts (+=)
 * weight * dL/dverts.  Edges with a zero-length edge vector or a degenerate face are skipped. */
int blur_smooth_loss_grad(const float *verts, int V, const void *topo, float weight, float *loss, float *grad_verts,
                          blur_stream_t stream);

/* Adam ("following SoftRas": lr 0.01, betas (0.5, 0.99); eps 1e-8), in place on n
 * parameters: m = b1 m + (1-b1) g; v = b2 v + (1-b2) g^2; p -= lr (m / (1-b1^step)) /
 * (sqrt(v / (1-b2^step)) + eps).  step is 1-based. */
int blur_adam_step(float *params, const float *grads, float *m, float *v, int64_t n, int step, float lr, float beta1,
                   float beta2, float eps, blur_stream_t stream);

/* sum_sq[0] (device double, overwritten) = sum (a - b)^2 over n floats (PSNR = 10 log10(n / sum_sq)
 * for values in [0, 1]). */
int blur_sum_sq_diff(const float *a, const float *b, int64_t n, double *sum_sq, blur_stream_t stream);

/* 3D IoU on res^3 voxels: on the shared bounding cube of both meshes (1%
 * margin), a voxel centre is inside a mesh iff the +x ray from it (origin nudged by (1e-7 sqrt2,
 * 1e-7 sqrt3) voxels in (y, z)) crosses an odd number of faces.  Computed in fp64 with explicit
 * rounding, so occupancies are bit-identical to the fp64 CPU oracle.  counts (device u64 [2],
 * overwritten) = (|A and B|, |A or B|); scratch (device) >= blur_voxel_scratch_bytes(res). */
size_t blur_voxel_scratch_bytes(int res);
int blur_voxel_iou(const float *va, int Va, const int32_t *fa, int Fa, const float *vb, int Vb, const int32_t *fb,
                   int Fb, int res, void *scratch, size_t scratch_bytes, unsigned long long *counts,
                   blur_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* BLURRAST_OPTIM_H */
