"""One process per GPU: shard independent images, no collective inside the loop.

VDAMP images are independent problems (src/vdamp.py:153-197 has no
cross-image state), so a batch is split into contiguous slices, one per
rank; each rank runs the whole loop locally and the only collective is the
final gather of x_hat to rank 0 (NCCL over NVLink/NVSwitch on B200, gloo in
the CPU tests).  Parallel equals serial bitwise: every image's arithmetic
is independent of the batch it runs in (tests/test_gpu_dist.py, mirroring
the reference's tests/test_cli.py:166-171).
"""

from __future__ import annotations

import os


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous slice [lo, hi) of ``total`` items for ``rank`` (ceil split, last ranks may be short
    or empty)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    per = -(-total // world)
    lo = min(total, rank * per)
    return lo, min(total, lo + per)


def env_rank_world() -> tuple[int, int, int]:
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def gather_images(local, total: int, group=None, dst: int = 0):
    """Gather per-rank (b_r, H, W) tensors into (total, H, W) on rank ``dst`` (None elsewhere).

    One ``gather`` to ``dst`` of fixed-size padded buffers (ceil(total/world)
    images per rank): only the destination receives the batch, every other
    rank sends its slice once.  Works for NCCL and gloo.  A rank with an empty
    slice passes a (0, H, W) tensor."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    per = -(-total // world)
    H, W = local.shape[1], local.shape[2]
    if local.shape[0] == per:
        buf = local.contiguous()
    else:
        buf = torch.zeros((per, H, W), dtype=local.dtype, device=local.device)
        buf[: local.shape[0]] = local
    send = torch.view_as_real(buf) if buf.is_complex() else buf       # complex as (re, im) pairs
    parts = [torch.empty_like(send) for _ in range(world)] if rank == dst else None
    dist.gather(send, parts, dst=dst, group=group)
    if rank != dst:
        return None
    out = []
    for r in range(world):
        lo, hi = shard_range(total, r, world)
        part = torch.view_as_complex(parts[r]) if buf.is_complex() else parts[r]
        out.append(part[: hi - lo])
    return torch.cat(out, 0)


def run_sharded(ys, masks, pmap, noise_vars, scales, n_iters, ground_truths=None, *, precision="fp32",
                with_traces=False, device=None, reconstruct=None):
    """Reconstruct a batch across all ranks of the default process group.

    Every rank passes the full input lists; rank r reconstructs its slice on
    ``device`` (default: the current CUDA device) and rank 0 receives the
    gathered (B, H, W) x_hat (None on the other ranks).  With ``with_traces``
    rank 0 also receives every image's RunTrace (``dist.gather_object``) and
    the call returns ``(x_hat, traces)``.  More ranks than images is allowed:
    ranks with an empty slice skip the reconstruction and still take part in
    the gather.  ``reconstruct`` replaces :func:`vdamp.run_batch` (same
    signature; the CPU tests pass a stand-in to exercise the sharding)."""
    import torch
    import torch.distributed as dist
    if reconstruct is None:
        from .vdamp import run_batch as reconstruct
    rank, world = dist.get_rank(), dist.get_world_size()
    total = len(masks)
    if total < 1:
        raise ValueError("empty batch")
    lo, hi = shard_range(total, rank, world)
    if device is None:
        device = torch.cuda.current_device() if torch.cuda.is_available() else "cpu"
    H, W = masks[0].shape
    cdtype = torch.complex64 if precision == "fp32" else torch.complex128
    traces = []
    if hi > lo:
        gts = None if ground_truths is None else ground_truths[lo:hi]
        pm = pmap[lo:hi] if isinstance(pmap, (list, tuple)) else pmap
        x, traces = reconstruct(ys[lo:hi], masks[lo:hi], pm, noise_vars[lo:hi], scales, n_iters, gts,
                                precision=precision, device=device, return_tensor=True)
    else:
        tdev = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)
        x = torch.empty((0, H, W), dtype=cdtype, device=tdev)
    backend = dist.get_backend()
    xg = gather_images(x if backend != "gloo" else x.cpu(), total)
    if not with_traces:
        return xg
    allt = [None] * world if rank == 0 else None
    dist.gather_object(traces, allt, dst=0)
    if rank != 0:
        return None, None
    return xg, [t for part in allt for t in part]
