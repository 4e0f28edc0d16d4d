"""Multi-GPU plumbing: one process per GPU, torch.distributed for the
process group.  The data path stays in libckks:

* queries (independent ciphertexts) shard across ranks with no collective
  (``shard_range``), as the paper's data parallelism over examples;
* ciphertexts are summed across ranks by an all-gather of the u64 limbs (int64 view,
  bit-identical copy) followed by ``ckks_modadd_gathered`` -- NCCL has no modular
  reduction (north star), so the reduction is our kernel, not NCCL's.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced [start, stop) of `total` items for `rank` (sizes differ by <= 1)."""
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def gather_limbs(t: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather a contiguous limb tensor [count, n_polys, capacity, N] (int64 view of u64)
    into [world, count, n_polys, capacity, N] -- the layout ckks_modadd_gathered reads."""
    world = dist.get_world_size(group)
    out = torch.empty((world, *t.shape), dtype=t.dtype, device=t.device)
    if t.is_cuda:
        dist.all_gather_into_tensor(out.view(-1), t.contiguous().view(-1), group=group)
    else:  # gloo (CPU tests): list form
        parts = list(out.unbind(0))
        dist.all_gather(parts, t.contiguous(), group=group)
    return out


def allsum_ciphertexts(ctx, buf, group=None):
    """Sum `buf` (a ckks.Buf) over all ranks modulo q_i; result replaces buf on every rank."""
    g = gather_limbs(buf.t, group)
    return ctx.modadd_gathered(g, g.shape[0], buf)
