"""Public Python API of the B200 motion-blur rasterizer.

`BlurRenderer` owns the device workspace for one (mesh topology, cameras, motions, image size)
configuration and calls the C ABI; `blur_render` is the differentiable (torch.autograd) form.
All arithmetic runs in libblurrast's CUDA kernels; torch only provides device memory and streams.
"""
from __future__ import annotations

import os
from typing import Optional

import numpy as np
import torch

from . import _lib


class WorkspaceArena:
    """One device workspace shared by renderers that run one after another (ShardedStep's passes): it
    grows to the largest request, and a renderer re-uploads its host tables whenever the previous call
    on the arena came from another renderer."""

    def __init__(self, device="cuda"):
        self.device = torch.device(device)
        self.buf = None
        self.owner = None

    def view(self, nbytes: int) -> torch.Tensor:
        if self.buf is None or self.buf.numel() < nbytes:
            self.buf = None
            self.buf = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
            self.buf[:256].zero_()
            self.owner = None
        return self.buf[:nbytes]


def cache_bytes_per_image(H: int, W: int, n_sub: int, delta: float = 0.0) -> int:
    """Size of BLUR_CACHE_VISIBILITY for one image: 2 B (+4 B of soft products) per pixel of the
    16-pixel-padded image and sub-frame."""
    px = ((H + 15) // 16 * 16) * ((W + 15) // 16 * 16)
    return int(n_sub) * px * (6 if delta > 0 else 2)


class BlurRenderer:
    """Motion-blurred rendering of one mesh topology for a batch of B observed images.

    faces: int32 [F,3] (device tensor or array); motion: dict of per-image arrays (kind, vec,
    angle, pivot, n_sub, n_seg, rule); cams: float [B,11]; H, W: image size.
    sub_range: optional int [B,2] half-open sub-frame ranges (sub-frame sharding).
    """

    # BLUR_CACHE_VISIBILITY budget: the per-(pixel, sub-frame) winner index (2 B, +4 B of soft products)
    # is kept between the forward and the backward only when it fits (C4: 0.84 GB; C5: 34 GB -> off)
    CACHE_BUDGET_BYTES = int(os.environ.get("BLURRAST_CACHE_BUDGET_MB", "1024")) << 20
    # ... except that a single image always keeps it up to CACHE_IMAGE_BYTES (C5 with soft coverage: 1.6 GB
    # per image; without it K9 runs its two-pass product recompute: 3.5x slower on C5)
    CACHE_IMAGE_BYTES = 2 << 30

    def __init__(self, faces, motion: dict, cams, H: int, W: int, V: int, device="cuda",
                 sub_range=None, max_chunk: int = 0, bin_factor: float = 0.0, solver: int = 0,
                 delta: float = 0.0, soft_cut: float = 0.0, soft_exact: bool = False,
                 soft_bin_factor: float = 0.0, cache_visibility: Optional[bool] = None,
                 workspace: Optional[WorkspaceArena] = None):
        _lib.load()
        self.arena = workspace
        self.device = torch.device(device)
        self.faces = torch.as_tensor(np.asarray(faces.cpu() if torch.is_tensor(faces) else faces),
                                     dtype=torch.int32).contiguous().to(self.device)
        self.motion = motion
        self.cams_np = np.asarray(cams, dtype=np.float64).reshape(-1, 11)
        self.B = int(self.cams_np.shape[0])
        self.H, self.W, self.V = int(H), int(W), int(V)
        self.F = int(self.faces.shape[0])
        self.N = np.asarray(motion["n_sub"], dtype=np.int64)
        self._motions = _lib.make_motions(motion)
        self._cams = _lib.make_cams(self.cams_np)
        self._sub = _lib.make_sub_range(sub_range)
        self._tables_resident = False          # the schedule tables change with the ranges
        self.max_chunk = int(max_chunk)
        self.bin_factor = float(bin_factor)
        self.solver = int(solver)
        # soft background coverage (NEXT-1, Eq.10-15): delta > 0 enables it
        self.delta, self.soft_cut, self.soft_exact = float(delta), float(soft_cut), bool(soft_exact)
        self.soft_bin_factor = float(soft_bin_factor)
        # K4 leaves the per-(pixel, sub-frame) winner slot for K6 (BLUR_CACHE_VISIBILITY): None = on iff
        # its size (2 B, + 4 B with soft coverage, per pixel of a 16-pixel-padded image and sub-frame)
        # fits CACHE_BUDGET_BYTES; without it K6 recomputes the visibility (k6_raster_bwd_fx)
        if cache_visibility is None:
            need = sum(cache_bytes_per_image(self.H, self.W, n, self.delta) for n in self.N)
            cache_visibility = need <= (self.CACHE_IMAGE_BYTES if self.B == 1 else self.CACHE_BUDGET_BYTES)
        self.cache_flags = _lib.BLUR_CACHE_VISIBILITY if (cache_visibility and self.solver == 0) else 0
        self.auto_bins = bin_factor == 0.0 or (self.delta > 0 and soft_bin_factor == 0.0)
        self.n_forward = 0
        self._alloc(self.bin_factor, self.soft_bin_factor)

    def _cfg(self, flags=0, census=None, events=None, soft_events=None):
        # the host tables (schedule, poses, chunks) stay in this renderer's own workspace between calls
        # with the same arguments: after the first upload every call skips the host->device copy
        if self._tables_resident and (self.arena is None or self.arena.owner is self):
            flags |= _lib.BLUR_TABLES_RESIDENT
        return _lib.make_config(self.max_chunk, flags | self.cache_flags, self.bin_factor, census, events, self.solver,
                                self.delta,
                                self.soft_cut, self.soft_exact, self.soft_bin_factor, soft_events)

    def _alloc(self, factor: float, soft_factor: float = 0.0):
        self.bin_factor = float(factor)
        self.soft_bin_factor = float(soft_factor)
        self._tables_resident = False
        cfg = self._cfg()
        self.ws_bytes = _lib.blur_workspace_bytes(self.V, self.F, self.B, self.H, self.W, self._motions,
                                                  self._cams, self._sub, cfg)
        self._ws = None
        if self.arena is None:
            self._ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=self.device)
            self._ws[:256].zero_()
        else:
            self.arena.view(self.ws_bytes)
        self._tables_resident = False

    @property
    def ws(self) -> torch.Tensor:
        """The workspace (own, or this renderer's view of a shared arena)."""
        return self._ws if self.arena is None else self.arena.view(self.ws_bytes)

    def _mark(self):
        self._tables_resident = True
        if self.arena is not None:
            self.arena.owner = self

    def _autosize(self, verts, colors, out, ids, ids_subframe, census, stream, events, soft_events):
        """First forward: if a binning needed more entries than the default capacity, grow the
        workspace (factor x needed/capacity, +25%) and render again (one synchronisation, once)."""
        self.auto_bins = False
        need, cap = _lib.blur_read_bins(self.ws, stream)
        sneed, scap = _lib.blur_read_soft_bins(self.ws, stream) if self.delta > 0 else (0, 0)
        if (need <= cap and sneed <= scap) or self.F == 0:
            return out
        base = self.bin_factor if self.bin_factor > 0 else 3.0
        sbase = self.soft_bin_factor if self.soft_bin_factor > 0 else 12.0
        self._alloc(base * need / max(cap, 1) * 1.25 if need > cap else base,
                    sbase * sneed / max(scap, 1) * 1.25 if sneed > scap else sbase)
        if census is not None:
            census.zero_()
        return self.forward(verts, colors, out, ids, ids_subframe, census, stream, events, soft_events)

    def set_sub_range(self, sub_range):
        """Per-image half-open sub-frame ranges for the next calls (None = all sub-frames).  The
        workspace was sized for the ranges given at construction; narrower ranges (e.g. [0, 0) for the
        views outside an optimisation batch) fit in it."""
        self._sub = _lib.make_sub_range(sub_range)
        self._tables_resident = False          # the schedule tables change with the ranges

    # -- forward / backward -------------------------------------------------------------
    def forward(self, verts: torch.Tensor, colors: torch.Tensor, out: Optional[torch.Tensor] = None,
                ids: Optional[torch.Tensor] = None, ids_subframe: int = -1, census: Optional[torch.Tensor] = None,
                stream=None, events=None, soft_events=None) -> torch.Tensor:
        self.n_forward += 1     # the workspace now holds this call's setup (see _BlurFn.backward)
        if out is None:
            out = torch.empty((self.B, self.H, self.W, 4), dtype=torch.float32, device=self.device)
        cfg = self._cfg(0, census, events, soft_events)
        _lib.blur_render_fwd(verts, self.faces, colors, self._motions, self._cams, self.B, self.H, self.W, out,
                             self.ws, sub_range=self._sub, ids=ids, ids_subframe=ids_subframe, cfg=cfg,
                             stream=stream)
        self._mark()
        if self.auto_bins:
            return self._autosize(verts, colors, out, ids, ids_subframe, census, stream, events, soft_events)
        return out

    def backward(self, verts: torch.Tensor, colors: torch.Tensor, grad_rgba: torch.Tensor, reuse_setup: bool = False,
                 grad_verts: Optional[torch.Tensor] = None, grad_colors: Optional[torch.Tensor] = None, stream=None,
                 events=None, soft_events=None):
        if grad_verts is None:
            grad_verts = torch.empty((self.V, 3), dtype=torch.float32, device=self.device)
        if grad_colors is None:
            grad_colors = torch.empty((self.V, 3), dtype=torch.float32, device=self.device)
        cfg = self._cfg(_lib.BLUR_REUSE_SETUP if reuse_setup else 0, events=events, soft_events=soft_events)
        _lib.blur_render_bwd(verts, self.faces, colors, self._motions, self._cams, self.B, self.H, self.W,
                             grad_rgba.contiguous(), grad_verts, grad_colors, self.ws, sub_range=self._sub, cfg=cfg,
                             stream=stream)
        self._mark()
        return grad_verts, grad_colors

    def l2_loss_grad(self, out: torch.Tensor, target: torch.Tensor, n_norm: int = 0, loss=None, grad=None,
                     stream=None):
        if loss is None:
            loss = torch.empty(1, dtype=torch.float32, device=self.device)
        if grad is None:
            grad = torch.empty_like(out)
        _lib.blur_l2_loss_grad(out, target, loss, grad, n_norm=n_norm, stream=stream)
        return loss, grad

    def status(self) -> int:
        return _lib.blur_read_status(self.ws)

    def capture_step(self, verts: torch.Tensor, colors: torch.Tensor, target: torch.Tensor, n_norm: int = 0):
        """CUDA-graph form of step() for launch-bound configurations (C1-C3: tens of microseconds of
        kernels per step).  One eager step sizes the workspace and leaves the host tables on the
        device; the graph then replays fwd -> L2 -> bwd on the given buffers (update them in place
        between replays).  Returns a StepGraph; its replay() enqueues the step on the current stream."""
        self.step(verts, colors, target, n_norm)             # eager: bins sized, tables resident
        torch.cuda.synchronize(self.device)
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream(device=self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                out = torch.empty((self.B, self.H, self.W, 4), dtype=torch.float32, device=self.device)
                cfg = self._cfg(_lib.BLUR_TABLES_RESIDENT)
                _lib.blur_render_fwd(verts, self.faces, colors, self._motions, self._cams, self.B, self.H, self.W,
                                     out, self.ws, sub_range=self._sub, cfg=cfg, stream=s)
                loss, grad = self.l2_loss_grad(out, target, n_norm=n_norm, stream=s)
                dv, dc = self.backward(verts, colors, grad, reuse_setup=True, stream=s)
        torch.cuda.current_stream(self.device).wait_stream(s)
        return StepGraph(g, loss, dv, dc, out)

    def step(self, verts, colors, target, n_norm: int = 0):
        """One inverse-rendering step: fwd -> L2 loss -> bwd (setup reused).  Device tensors in,
        (loss [1], dverts, dcolors, out) device tensors out."""
        out = self.forward(verts, colors)
        loss, g = self.l2_loss_grad(out, target, n_norm=n_norm)
        dv, dc = self.backward(verts, colors, g, reuse_setup=True)
        return loss, dv, dc, out


class StepGraph:
    """A captured fwd -> L2 -> bwd step (BlurRenderer.capture_step): replay() re-runs it on the buffers
    it was captured with; loss, dv, dc, out are the graph's output tensors."""

    def __init__(self, graph, loss, dv, dc, out):
        self.graph, self.loss, self.dv, self.dc, self.out = graph, loss, dv, dc, out

    def replay(self):
        self.graph.replay()
        return self.loss, self.dv, self.dc, self.out


class _BlurFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, verts, colors, renderer: BlurRenderer):
        out = renderer.forward(verts.contiguous(), colors.contiguous())
        ctx.renderer = renderer
        ctx.stamp = renderer.n_forward     # the forward whose setup (and visibility cache) the workspace holds
        ctx.save_for_backward(verts, colors)
        return out

    @staticmethod
    def backward(ctx, grad_out):
        verts, colors = ctx.saved_tensors
        # reuse the workspace's keyframes / coefficients / bins (and visibility cache) only if no other
        # forward ran on this renderer since this one; otherwise the backward rebuilds its own setup
        reuse = ctx.renderer.n_forward == ctx.stamp
        dv, dc = ctx.renderer.backward(verts.contiguous(), colors.contiguous(), grad_out.contiguous(),
                                       reuse_setup=reuse)
        return dv, dc, None


def blur_render(verts: torch.Tensor, colors: torch.Tensor, renderer: BlurRenderer) -> torch.Tensor:
    """Differentiable blurred render (B,H,W,4) of `verts` [V,3] / `colors` [V,3]."""
    return _BlurFn.apply(verts, colors, renderer)
