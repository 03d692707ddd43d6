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
    """

    def __init__(self, n_sub: Sequence[int], targets: torch.Tensor, make_renderer: Callable, rank: int,
                 world: int, split: int = 0, device="cpu", reduce: bool = None):
        self.rank, self.world = rank, world
        self.reduce = (world > 1) if reduce is None else reduce
        self.parts = partition(n_sub, world, split)
        self.mine = self.parts[rank]
        self.images = [u.image for u in self.mine]
        assert len(set(self.images)) == len(self.images), "one sub-frame range per image and rank"
        B = len(n_sub)
        self.n_norm = int(B * int(np.prod(targets.shape[1:])))        # mean over the whole batch
        self.targets = targets[self.images].contiguous() if self.images else targets[:0]
        self.renderer = make_renderer(self.images, [[u.k0, u.k1] for u in self.mine]) if self.images else None
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
        events: optional dict of CUDA event pairs recorded around the raster kernels ("fwd", "bwd",
        "soft_fwd", "soft_bwd"; see BlurRenderer.forward / backward)."""
        ev = events or {}
        V = verts.shape[0]
        if self.renderer is not None:
            if ev:
                out = self.renderer.forward(verts, colors, events=ev.get("fwd"), soft_events=ev.get("soft_fwd"))
            else:
                out = self.renderer.forward(verts, colors)
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
            if ev:
                dv, dc = self.renderer.backward(verts, colors, grads, reuse_setup=True, events=ev.get("bwd"),
                                                soft_events=ev.get("soft_bwd"))
            else:
                dv, dc = self.renderer.backward(verts, colors, grads, reuse_setup=True)
            flat = torch.cat([dv.reshape(-1), dc.reshape(-1), loss_all])
        else:
            flat = torch.zeros(6 * V + 1, dtype=verts.dtype, device=self.device)
        if self.reduce:
            dist.all_reduce(flat)
        return flat[-1:], flat[:3 * V].reshape(V, 3), flat[3 * V:6 * V].reshape(V, 3)
