"""Multi-process (gloo, world_size 2-3, CPU) checks of the image sharding and the final gather
used by bench.py / dist.run_sharded (no collective inside the VDAMP loop)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1911_01234_b200.dist import gather_images, run_sharded, shard_range


def test_shard_range_covers_batch():
    for total in (1, 7, 64, 65, 1024):
        for world in (1, 2, 3, 4, 8):
            got = [shard_range(total, r, world) for r in range(world)]
            covered = [i for lo, hi in got for i in range(lo, hi)]
            assert covered == list(range(total))
            assert max(hi - lo for lo, hi in got) == -(-total // world)
    assert shard_range(6, 3, 4) == (6, 6)             # empty slice for the last rank
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, total, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard_range(total, rank, world)
    # stand-in for each rank's reconstruction: image b is filled with b + 1j*b
    local = torch.stack([torch.full((4, 8), complex(b, -b), dtype=torch.complex64) for b in range(lo, hi)]) \
        if hi > lo else torch.empty((0, 4, 8), dtype=torch.complex64)
    out = gather_images(local, total)
    if rank == 0:
        q.put([complex(out[b, 0, 0]) for b in range(out.shape[0])])
    else:
        assert out is None
    dist.destroy_process_group()


def _spawn(target, world, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port) + args + (q,)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=60)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("total,world", [(5, 2), (8, 2), (1, 2), (4, 3)])
def test_gather_images(total, world):
    res = _spawn(_worker, world, total)
    assert res == [complex(b, -b) for b in range(total)]


class _Mask:
    def __init__(self, b):
        self.shape = (4, 8)
        self.b = b


class _Trace:
    def __init__(self, b):
        self.b = b


def _fake_reconstruct(ys, masks, pmap, noise_vars, scales, n_iters, gts, *, precision, device, return_tensor):
    """Stand-in for vdamp.run_batch: x_hat of image b is b * (1 + 2j) + n_iters."""
    assert return_tensor and precision == "fp32"
    x = torch.stack([torch.full((4, 8), complex(m.b + n_iters, 2 * m.b), dtype=torch.complex64) for m in masks])
    return x, [_Trace(m.b) for m in masks]


def _sharded_worker(rank, world, port, total, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    masks = [_Mask(b) for b in range(total)]
    x, traces = run_sharded([None] * total, masks, None, np.zeros(total), 2, 3, precision="fp32",
                            with_traces=True, device="cpu", reconstruct=_fake_reconstruct)
    if rank == 0:
        q.put(([complex(x[b, 0, 0]) for b in range(x.shape[0])], [t.b for t in traces]))
    else:
        assert x is None and traces is None
    dist.destroy_process_group()


@pytest.mark.parametrize("total,world", [(5, 2), (2, 3), (6, 4)])
def test_run_sharded_gloo(total, world):
    """run_sharded with more ranks than a ceil split fills (empty slices on the last ranks,
    ADVICE r1: must not deadlock) gathers every image and every trace in batch order."""
    xs, tb = _spawn(_sharded_worker, world, total)
    assert xs == [complex(b + 3, 2 * b) for b in range(total)]
    assert tb == list(range(total))
