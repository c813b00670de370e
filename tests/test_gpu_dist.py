"""Parallel equals serial bitwise (reference tests/test_cli.py:166-171): dist.run_sharded over
2 and 3 ranks (gloo, every rank on cuda:0 -- one GPU in this harness) against one process's
run_batch, images and traces.  The ranks do not wait on one another inside the loop (the only
collective is the final gather), so sharing one GPU changes nothing but the timing."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOTAL = 5


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    from paper_1911_01234_b200 import workload
    from paper_1911_01234_b200.dist import run_sharded
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w = workload.make_workload("cfg1", batch=TOTAL)
    x, tr = run_sharded(w.ys, w.masks, w.pmap, w.noise_vars, 4, 6, w.x0, precision="fp32", with_traces=True)
    if rank == 0:
        q.put((x.cpu().numpy(), [t.nmse_curve() for t in tr], [np.array([r.thresholds for r in t.records]) for t in tr]))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_run_sharded_equals_run_batch(world):
    import torch.multiprocessing as mp
    from paper_1911_01234_b200 import vdamp, workload
    w = workload.make_workload("cfg1", batch=TOTAL)
    xs, trs = vdamp.run_batch(w.ys, w.masks, w.pmap, w.noise_vars, 4, 6, w.x0, precision="fp32")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    x, nm, thr = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert x.shape == xs.shape
    assert np.array_equal(x.astype(np.complex128), xs)
    for b in range(TOTAL):
        assert np.array_equal(nm[b], trs[b].nmse_curve())
        assert np.array_equal(thr[b], np.array([r.thresholds for r in trs[b].records]))
