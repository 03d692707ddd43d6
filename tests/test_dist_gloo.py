"""Multi-process (world_size 2, gloo, CPU) tests of the sharding logic in paper_2602_07860_b200/dist.py.

The CUDA renderer is replaced by a CPU stand-in built on the fp64 oracle (test infrastructure), so
these tests check the partition, the partial-image all-reduce of sub-frame-split images, the
loss normalisation and the [dV || dC] all-reduce: the sharded step must equal the unsharded one.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import scenes
from paper_2602_07860_b200.dist import partition, split_groups, ShardedStep


class OracleRenderer:
    """CPU stand-in with the BlurRenderer interface (float64 torch tensors)."""

    def __init__(self, sc, images, sub_range):
        self.sc = sc.subset(images)
        self.sub = np.asarray(sub_range, np.int32)

    def forward(self, verts, colors, **kw):
        r = oracle.render_fwd(self.sc, sub_range=self.sub, threads=1, verts=verts.numpy(), colors=colors.numpy())
        return torch.from_numpy(r["rgba"])

    def l2_loss_grad(self, out, target, n_norm=0):
        n = n_norm if n_norm > 0 else out.numel()
        d = out - target
        return (d * d).sum().reshape(1) / n, 2.0 * d / n

    def backward(self, verts, colors, grad, reuse_setup=True, **kw):
        dv, dc = oracle.render_bwd(self.sc, grad.numpy(), sub_range=self.sub, threads=1, verts=verts.numpy(),
                                   colors=colors.numpy())
        return torch.from_numpy(dv), torch.from_numpy(dc)


def _scene(B):
    sc = scenes.random_mesh_scene(12, 3, H=12, W=14, B=B, motion=scenes.translate((0.5, 0.2, 0.1), N=6))
    sc.motion["n_sub"][:] = 6
    return sc


def _reference(sc):
    step = ShardedStep(sc.motion["n_sub"], torch.tensor(sc.target, dtype=torch.float64),
                       lambda im, sr: OracleRenderer(sc, im, sr), 0, 1)
    return step(torch.tensor(sc.verts, dtype=torch.float64), torch.tensor(sc.colors, dtype=torch.float64))


def _worker(rank, world, port, B, split, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sc = _scene(B)
    step = ShardedStep(sc.motion["n_sub"], torch.tensor(sc.target, dtype=torch.float64),
                       lambda im, sr: OracleRenderer(sc, im, sr), rank, world, split=split)
    loss, dv, dc = step(torch.tensor(sc.verts, dtype=torch.float64), torch.tensor(sc.colors, dtype=torch.float64))
    q.put((rank, loss.numpy().copy(), dv.numpy().copy(), dc.numpy().copy(), len(step.groups)))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(B, split, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, B, split, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(res, key=lambda x: x[0])


def test_partition_rules():
    parts = partition([10] * 16, 8)
    assert [len(p) for p in parts] == [2] * 8
    assert sorted(u.image for p in parts for u in p) == list(range(16))
    parts = partition([50], 4)                        # one image, four sub-frame ranges
    assert [(u.k0, u.k1) for p in parts for u in p] == [(0, 12), (12, 25), (25, 38), (38, 50)]
    assert split_groups(parts) == [(0, [0, 1, 2, 3])]
    parts = partition([100] * 64, 8, split=2)         # 2-D split
    assert sum(len(p) for p in parts) == 128
    assert all(len(rs) == 2 for _, rs in split_groups(parts))


@pytest.mark.parametrize("B,split", [(4, 0), (1, 0), (3, 2), (2, 4)])
def test_sharded_step_equals_single_process(B, split):
    """world 2; split 4 > world is clamped to 2 (one sub-frame range per image and rank)."""
    ref_loss, ref_dv, ref_dc = [t.numpy() for t in _reference(_scene(B))]
    res = _run(B, split)
    for rank, loss, dv, dc, ngroups in res:
        assert np.allclose(loss, ref_loss, rtol=1e-12, atol=1e-15)
        assert np.allclose(dv, ref_dv, rtol=1e-10, atol=1e-13)
        assert np.allclose(dc, ref_dc, rtol=1e-10, atol=1e-13)
    if B == 1 or split >= 2:
        # every split image is shared by ranks {0, 1}: one group, all its images in one all-reduce
        assert all(r[4] == 1 for r in res)


def test_split_at_world_one_is_the_unsplit_step():
    """world 1 with split 2: clamped to one range per image, equal to the plain step."""
    sc = _scene(2)
    ref = [t.numpy() for t in _reference(sc)]
    step = ShardedStep(sc.motion["n_sub"], torch.tensor(sc.target, dtype=torch.float64),
                       lambda im, sr: OracleRenderer(sc, im, sr), 0, 1, split=2)
    assert [(u.k0, u.k1) for u in step.mine] == [(0, 6), (0, 6)] and not step.groups
    got = [t.numpy() for t in step(torch.tensor(sc.verts, dtype=torch.float64),
                                   torch.tensor(sc.colors, dtype=torch.float64))]
    for a, b in zip(got, ref):
        assert np.array_equal(a, b)


def test_partition_split_clamped_and_groups_per_rank_set():
    parts = partition([6] * 4, 2, split=4)
    assert all(len({u.image for u in p}) == len(p) for p in parts)      # one range per image and rank
    assert [(u.k0, u.k1) for u in parts[0]] == [(0, 3)] * 4 and [(u.k0, u.k1) for u in parts[1]] == [(3, 6)] * 4
    assert {tuple(rs) for _, rs in split_groups(parts)} == {(0, 1)}
