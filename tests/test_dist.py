"""Multi-process (gloo, world_size 2, CPU) checks of the image sharding and the final gather
used by bench.py / dist.run_sharded (no collective inside the VDAMP loop)."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1911_01234_b200.dist import gather_images, shard_range


def test_shard_range_covers_batch():
    for total in (1, 7, 64, 65, 1024):
        for world in (1, 2, 3, 4, 8):
            got = [shard_range(total, r, world) for r in range(world)]
            covered = [i for lo, hi in got for i in range(lo, hi)]
            assert covered == list(range(total))
            assert max(hi - lo for lo, hi in got) == -(-total // world)
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
    dist.destroy_process_group()


@pytest.mark.parametrize("total", [5, 8])
def test_gather_images_two_ranks(total):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, total, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert res == [complex(b, -b) for b in range(total)]
