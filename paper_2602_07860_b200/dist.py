"""Multi-GPU sharding of the inverse-rendering step: one process per GPU.

Units of work are (image, k0, k1) sub-frame ranges.  Images are dealt round-robin to ranks
(image-major; consecutive images alternate translational / rotational views so ranks stay
balanced).  When there are fewer images than ranks, or when `split` > 1 is requested, every image
is cut into `split` contiguous sub-frame ranges owned by consecutive ranks ("sub-frame range"
sharding); those co-owners all-reduce their partial RGBA images (the blurred image is a sum over
sub-frames) before the loss.  After the backward pass one all-reduce of [dV || dC || loss]
(V x 6 + 1 fp32) sums the vertex gradients (torch.distributed: NCCL over NVLink on GPUs -- also at
world size 1, so the product path is the same at every scale -- gloo on the CPU tests).

Scale run (8 GPUs of one node, C5 cut into 2 sub-frame halves per image):
    torchrun --nnodes 1 --nproc-per-node 8 --master-addr 127.0.0.1 bench.py --gpus 8 --config C5 --split 2

The renderer is injected (`make_renderer`), so the same step logic runs with the CUDA renderer
on GPUs and with a CPU stand-in in the gloo tests.
"""
from __future__ import annotations

import dataclasses
from typing import Callable, Dict, List, Sequence, Tuple

import numpy as np
import torch
import torch.distributed as dist


@dataclasses.dataclass
class Unit:
    image: int
    k0: int
    k1: int


def partition(n_sub: Sequence[int], world: int, split: int = 0) -> List[List[Unit]]:
    """Work list per rank.  split = 0: automatic (1 if B >= world, else ceil(world / B)); a split
    above the world size is clamped to it, so that every rank holds at most one sub-frame range of
    an image (its renderer has one slot per image)."""
    B = len(n_sub)
    if world < 1:
        raise ValueError("world must be >= 1")
    if split <= 0:
        split = 1 if B >= world else -(-world // max(B, 1))
    split = min(split, world)
    units: List[Unit] = []
    for b in range(B):
        N = int(n_sub[b])
        parts = max(1, min(split, N))
        edges = [round(N * p / parts) for p in range(parts + 1)]
        for p in range(parts):
            units.append(Unit(b, edges[p], edges[p + 1]))
    # unit i -> rank i mod world: the parts of an image (consecutive units, at most `world` of them)
    # land on distinct, consecutive ranks
    out: List[List[Unit]] = [[] for _ in range(world)]
    for i, u in enumerate(units):
        out[i % world].append(u)
    return out


def split_groups(parts: List[List[Unit]]) -> List[Tuple[int, List[int]]]:
    """(image, ranks) for every image owned by more than one rank."""
    owners: Dict[int, set] = {}
    for r, us in enumerate(parts):
        for u in us:
            owners.setdefault(u.image, set()).add(r)
    return [(b, sorted(rs)) for b, rs in sorted(owners.items()) if len(rs) > 1]


class ShardedStep:
    """One rank's share of the step: fwd -> (partial-image all-reduce) -> L2 loss -> bwd ->
    all-reduce of [dV || dC || loss].

    make_renderer(images, sub_range) must return an object with forward(verts, colors) -> [b,H,W,4],
    l2_loss_grad(out, target, n_norm) -> (loss[1], grad) and
    backward(verts, colors, grad, reuse_setup=True) -> (dV, dC), all on `device`.
    reduce: run the collectives even at world size 1 (the bench does, so that NCCL is exercised).
    pass_images: when > 0 and smaller than this rank's image count (and no image is split), the rank
    runs its images in passes of that many -- fwd -> loss -> bwd per pass, gradients summed -- with
    renderers made as make_renderer(images, sub_range, workspace=arena) that share one workspace, so
    that the backward's per-(pixel, sub-frame) winner index of a pass fits a memory budget
    (BlurRenderer.CACHE_BUDGET_BYTES; cache_bytes_per_image).
    """

    def __init__(self, n_sub: Sequence[int], targets: torch.Tensor, make_renderer: Callable, rank: int,
                 world: int, split: int = 0, device="cpu", reduce: bool = None, pass_images: int = 0):
        self.rank, self.world = rank, world
        self.reduce = (world > 1) if reduce is None else reduce
        self.parts = partition(n_sub, world, split)
        self.mine = self.parts[rank]
        self.images = [u.image for u in self.mine]
        assert len(set(self.images)) == len(self.images), "one sub-frame range per image and rank"
        B = len(n_sub)
        self.n_norm = int(B * int(np.prod(targets.shape[1:])))        # mean over the whole batch
        self.targets = targets[self.images].contiguous() if self.images else targets[:0]
        whole = all(u.k0 == 0 and u.k1 == int(n_sub[u.image]) for u in self.mine)
        npass = len(self.images) if not (0 < pass_images < len(self.images) and whole) else pass_images
        self.passes = [list(range(i, min(i + npass, len(self.images)))) for i in range(0, len(self.images), max(npass, 1))]
        if len(self.passes) > 1:
            from .renderer import WorkspaceArena
            arena = WorkspaceArena(device)
            self.renderers = [make_renderer([self.images[i] for i in p], [[self.mine[i].k0, self.mine[i].k1] for i in p],
                                            workspace=arena) for p in self.passes]
        else:
            self.renderers = [make_renderer(self.images, [[u.k0, u.k1] for u in self.mine])] if self.images else []
        self.renderer = self.renderers[0] if self.renderers else None
        # loss is counted once per image: by the co-owner holding k0 == 0
        self.loss_mask = torch.tensor([1.0 if u.k0 == 0 else 0.0 for u in self.mine], dtype=targets.dtype,
                                      device=device)
        self.device = device
        # one process group per distinct set of co-owning ranks; every rank creates every group, in
        # the same order (torch.distributed requires it); this rank keeps the slots of its images
        self.groups: List[Tuple[torch.Tensor, object]] = []
        if world > 1:
            sets: Dict[Tuple[int, ...], List[int]] = {}
            for b, ranks in split_groups(self.parts):
                sets.setdefault(tuple(ranks), []).append(b)
            for ranks, imgs in sorted(sets.items()):
                g = dist.new_group(list(ranks))
                if rank in ranks:
                    slots = torch.tensor([self.images.index(b) for b in imgs], dtype=torch.long, device=device)
                    self.groups.append((slots, g))

    @staticmethod
    def _pick(ev, key, p):
        """events[key] is a list of CUDA event pairs, one per pass (or None)."""
        e = ev.get(key)
        return e[p] if e else None

    @property
    def n_passes(self) -> int:
        return len(self.passes)

    def census(self, verts: torch.Tensor, colors: torch.Tensor, census: torch.Tensor) -> None:
        """Algorithmic unit counts of this rank's forward (summed over the passes) into `census`."""
        for r in self.renderers:
            r.forward(verts, colors, census=census)

    def _passes(self, verts, colors, targets_ready, ev):
        """Whole images in passes sharing one workspace: fwd -> loss -> bwd per pass, sums accumulated."""
        V = verts.shape[0]
        dv = torch.zeros(V, 3, dtype=verts.dtype, device=self.device)
        dc = torch.zeros(V, 3, dtype=verts.dtype, device=self.device)
        loss = torch.zeros(1, dtype=verts.dtype, device=self.device)

        pick = self._pick
        for p, (slots, r) in enumerate(zip(self.passes, self.renderers)):
            out = r.forward(verts, colors, events=pick(ev, "fwd", p), soft_events=pick(ev, "soft_fwd", p))
            if p == 0 and targets_ready is not None:
                torch.cuda.current_stream().wait_event(targets_ready)
            tg = self.targets[slots[0]:slots[-1] + 1]
            lp, g = r.l2_loss_grad(out, tg, n_norm=self.n_norm)
            dvp, dcp = r.backward(verts, colors, g, reuse_setup=True, events=pick(ev, "bwd", p),
                                  soft_events=pick(ev, "soft_bwd", p))
            dv += dvp
            dc += dcp
            loss += lp
        flat = torch.cat([dv.reshape(-1), dc.reshape(-1), loss])
        if self.reduce:
            dist.all_reduce(flat)
        return flat[-1:], flat[:3 * V].reshape(V, 3), flat[3 * V:6 * V].reshape(V, 3)

    def reduce_partials(self, out: torch.Tensor) -> None:
        """Sum the partial images of the split images over their co-owners: one all-reduce per group
        of ranks, all of the group's images at once."""
        for slots, g in self.groups:
            part = out.index_select(0, slots)
            dist.all_reduce(part, group=g)
            out.index_copy_(0, slots, part)

    def __call__(self, verts: torch.Tensor, colors: torch.Tensor, targets_ready=None, events=None):
        """targets_ready: optional CUDA event after which self.targets is valid (a loader copying the
        next observed images on another stream overlaps that copy with the forward pass).
        events: optional dict ("fwd", "bwd", "soft_fwd", "soft_bwd") of lists of CUDA event pairs, one
        pair per pass, recorded around the raster kernels (see BlurRenderer.forward / backward)."""
        ev = events or {}
        V = verts.shape[0]
        if len(self.passes) > 1:
            return self._passes(verts, colors, targets_ready, ev)
        if self.renderer is not None:
            out = self.renderer.forward(verts, colors, events=self._pick(ev, "fwd", 0),
                                        soft_events=self._pick(ev, "soft_fwd", 0))
            if targets_ready is not None:
                torch.cuda.current_stream().wait_event(targets_ready)
            self.reduce_partials(out)
            if all(u.k0 == 0 for u in self.mine):                      # loss counted here for every image
                loss_all, grads = self.renderer.l2_loss_grad(out, self.targets, n_norm=self.n_norm)
            else:
                loss_all = torch.zeros(1, dtype=out.dtype, device=self.device)
                grads = torch.empty_like(out)
                for i in range(len(self.images)):
                    li, gi = self.renderer.l2_loss_grad(out[i:i + 1].contiguous(),
                                                        self.targets[i:i + 1].contiguous(), n_norm=self.n_norm)
                    loss_all += li * self.loss_mask[i]
                    grads[i].copy_(gi[0])
            dv, dc = self.renderer.backward(verts, colors, grads, reuse_setup=True, events=self._pick(ev, "bwd", 0),
                                            soft_events=self._pick(ev, "soft_bwd", 0))
            flat = torch.cat([dv.reshape(-1), dc.reshape(-1), loss_all])
        else:
            flat = torch.zeros(6 * V + 1, dtype=verts.dtype, device=self.device)
        if self.reduce:
            dist.all_reduce(flat)
        return flat[-1:], flat[:3 * V].reshape(V, 3), flat[3 * V:6 * V].reshape(V, 3)
