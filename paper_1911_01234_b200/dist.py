"""One process per GPU: shard independent images, no collective inside the loop.

VDAMP images are independent problems (src/vdamp.py:153-197 has no
cross-image state), so a batch is split into contiguous slices, one per
rank; each rank runs the whole loop locally and the only collective is the
final gather of x_hat to rank 0 (NCCL over NVLink/NVSwitch on B200, gloo in
the CPU tests).
"""

from __future__ import annotations

import os


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous slice [lo, hi) of ``total`` items for ``rank`` (ceil split, last ranks may be short)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    per = -(-total // world)
    lo = min(total, rank * per)
    return lo, min(total, lo + per)


def env_rank_world() -> tuple[int, int, int]:
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def gather_images(local, total: int, group=None):
    """Gather per-rank (b_r, H, W) complex tensors into (total, H, W) on rank 0 (None elsewhere).

    Uses all_gather on fixed-size padded real views (works for NCCL and gloo)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    per = -(-total // world)
    H, W = local.shape[1], local.shape[2]
    buf = torch.zeros((per, H, W), dtype=local.dtype, device=local.device)
    buf[: local.shape[0]] = local
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    if rank != 0:
        return None
    out = []
    for r in range(world):
        lo, hi = shard_range(total, r, world)
        out.append(parts[r][: hi - lo])
    return torch.cat(out, 0)


def run_sharded(ys, masks, pmap, noise_vars, scales, n_iters, *, precision="fp32"):
    """Reconstruct a batch across all ranks of the default process group.

    Every rank passes the full input lists; rank r reconstructs its slice on
    cuda:LOCAL_RANK and rank 0 receives the gathered (B, H, W) result."""
    import torch
    import torch.distributed as dist
    from .vdamp import run_batch
    rank, world = dist.get_rank(), dist.get_world_size()
    lo, hi = shard_range(len(masks), rank, world)
    dev = torch.cuda.current_device()
    x, _ = run_batch(ys[lo:hi], masks[lo:hi], pmap, noise_vars[lo:hi], scales, n_iters,
                     precision=precision, device=dev, return_tensor=True)
    return gather_images(x, len(masks))
