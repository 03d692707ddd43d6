"""Thin ctypes binding of libblurrast (include/blurrast.h): argument marshalling only.

Every function has the name of the C entry point it calls.  Device buffers are passed as torch
CUDA tensors (checked for device, dtype and contiguity), host structs are built from numpy arrays.
There is no CPU fallback: if libblurrast.so is missing or CUDA is unavailable the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BLURRAST_LIB") or os.path.join(_HERE, "libblurrast.so")   # override: A/B builds
_lock = threading.Lock()
_lib = None

BLUR_OK, BLUR_EINVAL, BLUR_EBEHIND, BLUR_ENOMEM, BLUR_ECUDA, BLUR_EOVERFLOW = range(6)
BLUR_ST_EINVAL, BLUR_ST_EBEHIND, BLUR_ST_EOVERFLOW, BLUR_ST_EINTERNAL = 1, 2, 4, 8
BLUR_REUSE_SETUP = 1
BLUR_CACHE_VISIBILITY = 2
BLUR_TABLES_RESIDENT = 4
STATUS_NAMES = {0: "BLUR_OK", 1: "BLUR_EINVAL", 2: "BLUR_EBEHIND", 3: "BLUR_ENOMEM", 4: "BLUR_ECUDA",
                5: "BLUR_EOVERFLOW"}

EXPORTED = ["blur_workspace_bytes", "blur_render_fwd", "blur_render_bwd", "blur_l2_loss_grad",
            "blur_read_status", "blur_read_bins", "blur_read_soft_bins", "blur_ffma_probe", "blur_last_error",
            "blur_abi_version",
            # include/blurrast_optim.h (NEXT-4 recovery step)
            "blur_topology_bytes", "blur_topology_build", "blur_l1_loss_grad", "blur_laplacian_loss_grad",
            "blur_smooth_loss_grad", "blur_adam_step", "blur_sum_sq_diff", "blur_voxel_scratch_bytes",
            "blur_voxel_iou"]
ABI_VERSION = 2


class BlurError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__("%s: %s" % (STATUS_NAMES.get(code, str(code)), msg))
        self.code = code


class blur_motion(C.Structure):
    _fields_ = [("kind", C.c_int32), ("vec", C.c_float * 3), ("angle", C.c_float), ("pivot", C.c_float * 3),
                ("n_subframes", C.c_int32), ("n_segments", C.c_int32), ("sched_rule", C.c_int32)]


class blur_camera(C.Structure):
    _fields_ = [("eye", C.c_float * 3), ("target", C.c_float * 3), ("up", C.c_float * 3),
                ("half_fov", C.c_float), ("z_near", C.c_float)]


class blur_config(C.Structure):
    _fields_ = [("max_chunk", C.c_int32), ("flags", C.c_int32), ("bin_factor", C.c_float),
                ("census", C.c_void_p), ("raster_events", C.c_void_p * 2), ("solver", C.c_int32),
                ("delta", C.c_float), ("soft_cut", C.c_float), ("soft_exact", C.c_int32),
                ("soft_bin_factor", C.c_float), ("soft_events", C.c_void_p * 2)]


def load():
    """Load libblurrast.so (fails loudly if it has not been built)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError("libblurrast.so not built (%s); run __graft_entry__.build()" % LIB_PATH)
        lib = C.CDLL(LIB_PATH)
        P, I, SZ = C.c_void_p, C.c_int, C.c_size_t
        lib.blur_workspace_bytes.argtypes = [I, I, I, I, I, P, P, P, P]
        lib.blur_workspace_bytes.restype = SZ
        lib.blur_render_fwd.argtypes = [P, I, P, I, P, P, P, I, I, I, P, P, P, I, P, P, SZ, P]
        lib.blur_render_bwd.argtypes = [P, I, P, I, P, P, P, I, I, I, P, P, P, P, P, P, SZ, P]
        lib.blur_l2_loss_grad.argtypes = [P, P, C.c_int64, C.c_int64, P, P, P]
        lib.blur_read_status.argtypes = [P, P, P]
        lib.blur_read_bins.argtypes = [P, P, P, P]
        lib.blur_read_soft_bins.argtypes = [P, P, P, P]
        lib.blur_ffma_probe.argtypes = [I, I, P, P, P]
        lib.blur_last_error.restype = C.c_char_p
        F, D = C.c_float, C.c_double
        lib.blur_topology_bytes.argtypes = [I, I, P]
        lib.blur_topology_bytes.restype = SZ
        lib.blur_topology_build.argtypes = [I, I, P, P, SZ, P]
        lib.blur_l1_loss_grad.argtypes = [P, P, I, I, I, P, I, P, P, P]
        lib.blur_laplacian_loss_grad.argtypes = [P, P, I, P, F, P, P, P]
        lib.blur_smooth_loss_grad.argtypes = [P, I, P, F, P, P, P]
        lib.blur_adam_step.argtypes = [P, P, P, P, C.c_int64, I, F, F, F, F, P]
        lib.blur_sum_sq_diff.argtypes = [P, P, C.c_int64, P, P]
        lib.blur_voxel_scratch_bytes.argtypes = [I]
        lib.blur_voxel_scratch_bytes.restype = SZ
        lib.blur_voxel_iou.argtypes = [P, I, P, I, P, I, P, I, I, P, SZ, P, P]
        lib.blur_abi_version.restype = I
        if lib.blur_abi_version() != ABI_VERSION:
            raise ImportError("libblurrast.so ABI %d != binding ABI %d: rebuild" % (lib.blur_abi_version(), ABI_VERSION))
        _lib = lib
        return lib


def _check(code):
    if code != BLUR_OK:
        raise BlurError(code, load().blur_last_error().decode())
    return code


def _dev(t, dtype, name):
    import torch
    if t is None:
        return None
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError("%s must be a CUDA tensor" % name)
    if t.dtype != dtype:
        raise TypeError("%s must be %s, got %s" % (name, dtype, t.dtype))
    if not t.is_contiguous():
        raise ValueError("%s must be contiguous" % name)
    return C.c_void_p(t.data_ptr())


def _stream(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


# ------------------------------------------------------------------------- host structs

def make_motions(motion: dict):
    """motion dict of arrays (see scenes/) -> ctypes blur_motion[B]."""
    B = len(motion["kind"])
    arr = (blur_motion * max(B, 1))()
    for b in range(B):
        m = arr[b]
        m.kind = int(motion["kind"][b])
        m.vec[:] = [float(x) for x in motion["vec"][b]]
        m.angle = float(motion["angle"][b])
        m.pivot[:] = [float(x) for x in motion["pivot"][b]]
        m.n_subframes = int(motion["n_sub"][b])
        m.n_segments = int(motion["n_seg"][b])
        m.sched_rule = int(motion["rule"][b])
    return arr


def make_cams(cams: np.ndarray):
    """float [B,11] (eye, target, up, half_fov, z_near) -> ctypes blur_camera[B]."""
    cams = np.asarray(cams, dtype=np.float64)
    B = cams.shape[0]
    arr = (blur_camera * max(B, 1))()
    for b in range(B):
        c = arr[b]
        c.eye[:] = list(cams[b, 0:3])
        c.target[:] = list(cams[b, 3:6])
        c.up[:] = list(cams[b, 6:9])
        c.half_fov = float(cams[b, 9])
        c.z_near = float(cams[b, 10])
    return arr


def make_sub_range(sub_range):
    if sub_range is None:
        return None
    a = np.ascontiguousarray(np.asarray(sub_range, dtype=np.int32).reshape(-1, 2))
    return a


def make_config(max_chunk=0, flags=0, bin_factor=0.0, census=None, events=None, solver=0, delta=0.0,
                soft_cut=0.0, soft_exact=False, soft_bin_factor=0.0, soft_events=None):
    """events / soft_events: optional (torch.cuda.Event, torch.cuda.Event) recorded around the raster
    kernel / the soft-coverage kernel."""
    cfg = blur_config(int(max_chunk), int(flags), float(bin_factor),
                      None if census is None else C.c_void_p(census.data_ptr()))
    cfg.solver = int(solver)
    cfg.delta = float(delta)
    cfg.soft_cut = float(soft_cut)
    cfg.soft_exact = int(bool(soft_exact))
    cfg.soft_bin_factor = float(soft_bin_factor)
    if events is not None:
        cfg.raster_events[0] = events[0].cuda_event
        cfg.raster_events[1] = events[1].cuda_event
    if soft_events is not None:
        cfg.soft_events[0] = soft_events[0].cuda_event
        cfg.soft_events[1] = soft_events[1].cuda_event
    return cfg


def _np_ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _ref(x):
    return None if x is None else C.byref(x)


# ------------------------------------------------------------------------- entry points

def blur_workspace_bytes(V, F, B, H, W, motions, cams, sub_range=None, cfg=None) -> int:
    n = load().blur_workspace_bytes(V, F, B, H, W, motions, cams, _np_ptr(sub_range), _ref(cfg))
    if n == 0:
        raise BlurError(BLUR_EINVAL, load().blur_last_error().decode())
    return int(n)


def blur_render_fwd(verts, faces, colors, motions, cams, B, H, W, out_rgba, ws, sub_range=None, ids=None,
                    ids_subframe=-1, cfg=None, stream=None):
    import torch
    V = verts.shape[0]
    F = faces.shape[0]
    return _check(load().blur_render_fwd(
        _dev(verts, torch.float32, "verts"), V, _dev(faces, torch.int32, "faces"), F,
        _dev(colors, torch.float32, "colors"), motions, cams, B, H, W, _np_ptr(sub_range),
        _dev(out_rgba, torch.float32, "out_rgba"), _dev(ids, torch.int32, "ids"), int(ids_subframe),
        _ref(cfg), _dev(ws, torch.uint8, "ws"), ws.numel(), _stream(stream)))


def blur_render_bwd(verts, faces, colors, motions, cams, B, H, W, grad_rgba, grad_verts, grad_colors, ws,
                    sub_range=None, cfg=None, stream=None):
    import torch
    V = verts.shape[0]
    F = faces.shape[0]
    return _check(load().blur_render_bwd(
        _dev(verts, torch.float32, "verts"), V, _dev(faces, torch.int32, "faces"), F,
        _dev(colors, torch.float32, "colors"), motions, cams, B, H, W, _np_ptr(sub_range),
        _dev(grad_rgba, torch.float32, "grad_rgba"), _dev(grad_verts, torch.float32, "grad_verts"),
        _dev(grad_colors, torch.float32, "grad_colors"), _ref(cfg), _dev(ws, torch.uint8, "ws"), ws.numel(),
        _stream(stream)))


def blur_l2_loss_grad(out, target, loss, grad, n_norm=0, stream=None):
    import torch
    return _check(load().blur_l2_loss_grad(
        _dev(out, torch.float32, "out"), _dev(target, torch.float32, "target"), out.numel(), int(n_norm),
        _dev(loss, torch.float32, "loss"), _dev(grad, torch.float32, "grad"), _stream(stream)))


def blur_read_status(ws, stream=None) -> int:
    import torch
    st = C.c_int32(0)
    _check(load().blur_read_status(_dev(ws, torch.uint8, "ws"), _stream(stream), C.byref(st)))
    return int(st.value)


def blur_read_bins(ws, stream=None):
    """(entries needed by the last binning, entry capacity of the workspace); synchronises."""
    import torch
    need, cap = C.c_longlong(0), C.c_longlong(0)
    _check(load().blur_read_bins(_dev(ws, torch.uint8, "ws"), _stream(stream), C.byref(need), C.byref(cap)))
    return int(need.value), int(cap.value)


def blur_read_soft_bins(ws, stream=None):
    """The same for the soft-coverage bins (0, 0 when delta == 0); synchronises."""
    import torch
    need, cap = C.c_longlong(0), C.c_longlong(0)
    _check(load().blur_read_soft_bins(_dev(ws, torch.uint8, "ws"), _stream(stream), C.byref(need), C.byref(cap)))
    return int(need.value), int(cap.value)


def blur_ffma_probe(ctas, iters, sink, stream=None) -> float:
    import torch
    fl = C.c_double(0)
    _check(load().blur_ffma_probe(int(ctas), int(iters), _dev(sink, torch.float32, "sink"), C.byref(fl),
                                  _stream(stream)))
    return float(fl.value)


def blur_last_error() -> str:
    return load().blur_last_error().decode()


def blur_abi_version() -> int:
    return int(load().blur_abi_version())


# ------------------------------------------------------------------------- recovery step (blurrast_optim.h)

def blur_topology_bytes(V, faces_np) -> int:
    f = np.ascontiguousarray(np.asarray(faces_np, dtype=np.int32).reshape(-1, 3))
    n = load().blur_topology_bytes(int(V), f.shape[0], _np_ptr(f))
    if n == 0:
        raise BlurError(BLUR_EINVAL, load().blur_last_error().decode())
    return int(n)


def blur_topology_build(V, faces_np, topo, stream=None):
    import torch
    f = np.ascontiguousarray(np.asarray(faces_np, dtype=np.int32).reshape(-1, 3))
    return _check(load().blur_topology_build(int(V), f.shape[0], _np_ptr(f), _dev(topo, torch.uint8, "topo"),
                                             topo.numel(), _stream(stream)))


def blur_l1_loss_grad(out, target, loss, grad, image_mask=None, n_images=0, stream=None):
    import torch
    B, H, W = out.shape[0], out.shape[1], out.shape[2]
    return _check(load().blur_l1_loss_grad(
        _dev(out, torch.float32, "out"), _dev(target, torch.float32, "target"), B, H, W,
        _dev(image_mask, torch.uint8, "image_mask"), int(n_images), _dev(loss, torch.float32, "loss"),
        _dev(grad, torch.float32, "grad"), _stream(stream)))


def blur_laplacian_loss_grad(verts, verts0, topo, weight, loss, grad_verts, stream=None):
    import torch
    return _check(load().blur_laplacian_loss_grad(
        _dev(verts, torch.float32, "verts"), _dev(verts0, torch.float32, "verts0"), verts.shape[0],
        _dev(topo, torch.uint8, "topo"), float(weight), _dev(loss, torch.float32, "loss"),
        _dev(grad_verts, torch.float32, "grad_verts"), _stream(stream)))


def blur_smooth_loss_grad(verts, topo, weight, loss, grad_verts, stream=None):
    import torch
    return _check(load().blur_smooth_loss_grad(
        _dev(verts, torch.float32, "verts"), verts.shape[0], _dev(topo, torch.uint8, "topo"), float(weight),
        _dev(loss, torch.float32, "loss"), _dev(grad_verts, torch.float32, "grad_verts"), _stream(stream)))


def blur_adam_step(params, grads, m, v, step, lr=0.01, beta1=0.5, beta2=0.99, eps=1e-8, stream=None):
    import torch
    return _check(load().blur_adam_step(
        _dev(params, torch.float32, "params"), _dev(grads, torch.float32, "grads"), _dev(m, torch.float32, "m"),
        _dev(v, torch.float32, "v"), params.numel(), int(step), float(lr), float(beta1), float(beta2), float(eps),
        _stream(stream)))


def blur_sum_sq_diff(a, b, out, stream=None):
    import torch
    return _check(load().blur_sum_sq_diff(_dev(a, torch.float32, "a"), _dev(b, torch.float32, "b"), a.numel(),
                                          _dev(out, torch.float64, "out"), _stream(stream)))


def blur_voxel_scratch_bytes(res) -> int:
    return int(load().blur_voxel_scratch_bytes(int(res)))


def blur_voxel_iou(va, fa, vb, fb, res, scratch, counts, stream=None):
    import torch
    return _check(load().blur_voxel_iou(
        _dev(va, torch.float32, "va"), va.shape[0], _dev(fa, torch.int32, "fa"), fa.shape[0],
        _dev(vb, torch.float32, "vb"), vb.shape[0], _dev(fb, torch.int32, "fb"), fb.shape[0], int(res),
        _dev(scratch, torch.uint8, "scratch"), scratch.numel(), _dev(counts, torch.int64, "counts"),
        _stream(stream)))
