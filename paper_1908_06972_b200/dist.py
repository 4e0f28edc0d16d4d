"""Multi-GPU plumbing: one process per GPU, torch.distributed for the
process group.  The data path stays in libckks:

* queries (independent ciphertexts) shard across ranks with no collective
  (``shard_range``), as the paper's data parallelism over examples;
* ciphertexts are summed across ranks by an all-gather of the u64 limbs (int64 view,
  bit-identical copy) followed by ``ckks_modadd_gathered`` -- NCCL has no modular
  reduction (north star), so the reduction is our kernel, not NCCL's;
* limb-sharded key switching (``sharded_keyswitch``; row f3's digit-pipelined form
  ``pipelined_sharded_keyswitch`` overlaps the digit transfers with ModUp);
* or (row f3) by ``PeerModSum``: buffers mapped into every peer once through CUDA IPC, then
  one ``ckks_p2p_modsum`` kernel per rank reduces its slice straight out of the peers'
  memory and stores the sum into all of them (reduce-scatter + all-gather + mod-add fused).
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


class PeerModSum:
    """Fused peer-memory modular all-reduce of one registered ciphertext buffer (row f3).

    Registration (once): every rank exports its buffer's IPC handle, the handles are
    exchanged with ``all_gather_object`` over the process group, and each rank maps its
    peers' buffers.  ``__call__`` sums the buffer over ranks mod q_i in place:
    stream sync + barrier (inputs complete everywhere), one ckks_p2p_modsum kernel, stream
    sync + barrier (every rank's slice stored everywhere)."""

    def __init__(self, ctx, buf, group=None):
        self.ctx, self.buf, self.group = ctx, buf, group
        self.R = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        handle = ctx.ipc_export(buf.t)
        handles = [None] * self.R
        dist.all_gather_object(handles, handle, group=group)
        self.ptrs, self._opened = [], []
        for r, (h, off) in enumerate(handles):
            if r == self.rank:
                self.ptrs.append(buf.t.data_ptr())
            else:
                p = ctx.ipc_open(h, off)
                self._opened.append(p)
                self.ptrs.append(p)

    def _sync(self):
        if self.buf.t.is_cuda:
            torch.cuda.synchronize(self.buf.t.device)
        dist.barrier(group=self.group)

    def __call__(self):
        self._sync()  # every rank's input complete before any peer reads it
        self.ctx.p2p_modsum(self.ptrs, self.ptrs, self.rank, self.buf)
        self._sync()  # every rank's slice stored into every peer
        return self.buf

    def close(self):
        for p in self._opened:
            self.ctx.ipc_close(p)
        self._opened = []


# ---- limb-sharded key switch ---------------------------------------------------
def limb_shard(L: int, R: int, r: int, l: int | None = None) -> tuple[int, int, int]:
    """Rank r's limbs [lo, hi) at level l when the top level L is split in shards of
    w = ceil(L / R) limbs (ownership is fixed by global limb index, so no re-sharding is
    needed as rescales drop limbs).  Returns (lo, hi, w); hi <= lo means no limbs."""
    l = L if l is None else l
    w = -(-L // R)
    lo = r * w
    return lo, min(lo + w, l), w


class Transport:
    """Collectives used by the sharded path.  `Torch` uses torch.distributed (NCCL on GPU,
    gloo on CPU); tests may substitute an in-process emulation."""

    def __init__(self, group=None):
        self.group = group
        self.R = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def all_gather(self, t: torch.Tensor) -> torch.Tensor:
        out = torch.empty((self.R, *t.shape), dtype=t.dtype, device=t.device)
        if t.is_cuda:
            dist.all_gather_into_tensor(out.view(-1), t.contiguous().view(-1), group=self.group)
        else:
            dist.all_gather(list(out.unbind(0)), t.contiguous(), group=self.group)
        return out

    def broadcast(self, t: torch.Tensor, src: int) -> torch.Tensor:
        dist.broadcast(t, src=src, group=self.group)
        return t

    def broadcast_async(self, t: torch.Tensor, src: int):
        """Enqueue a broadcast; the handle's wait() orders the CURRENT stream after it (NCCL)
        or blocks until it is done (gloo) -- the host does not wait on GPU."""
        return dist.broadcast(t, src=src, group=self.group, async_op=True)


def sharded_keyswitch(ctx, tr: Transport, kind: int, step: int, a, b, L: int, l: int, out_alloc):
    """One limb-sharded key switch on this rank's shard `a` (and `b` for relinearisation):
    local digits -> all-gather -> ModUp/inner product/ModDown for the owned targets.
    Returns this rank's output shard (None if it owns no limbs at level l)."""
    lo, hi, w = limb_shard(L, tr.R, tr.rank, l)
    cnt = a.count if a is not None else 0
    D_own = torch.zeros((cnt, w, ctx.N), dtype=torch.int64, device=ctx.device)
    out = out_alloc(cnt, hi - lo) if hi > lo else None
    if hi > lo:
        ctx.shard_ks_digits(kind, step, a, b, lo, l, w, out, D_own)
    D_all = tr.all_gather(D_own)  # [R][count][w][N]
    if hi > lo:
        ctx.shard_ks_finish(kind, step, D_all, tr.R, w, a, lo, l, out)
    return out


def window_order(R: int, rank: int) -> list[int]:
    """Order in which a rank folds the digit windows in: its own first (no transfer), then the
    others in the order their broadcasts are enqueued."""
    return [rank] + [r for r in range(R) if r != rank]


def pipelined_sharded_keyswitch(ctx, tr: Transport, kind: int, step: int, a, b, L: int, l: int, out_alloc):
    """Digit-pipelined limb-sharded key switch (row f3): the R digit shards move as R
    broadcasts enqueued up front on the collective stream; this rank folds its own window in
    at once and each peer's window as soon as that broadcast has landed (the wait orders the
    compute stream after it), so the transfers overlap ModUp + inner product.  Bit-identical
    to sharded_keyswitch."""
    lo, hi, w = limb_shard(L, tr.R, tr.rank, l)
    cnt = a.count if a is not None else 0
    if a is None:  # a rank without limbs still serves its (empty) broadcast
        cnt = 0
    D_all = torch.zeros((tr.R, max(cnt, 1), w, ctx.N), dtype=torch.int64, device=ctx.device)
    out = out_alloc(cnt, hi - lo) if hi > lo else None
    if hi > lo:
        ctx.shard_ks_digits(kind, step, a, b, lo, l, w, out, D_all[tr.rank, :cnt])
    handles = {r: tr.broadcast_async(D_all[r], r) for r in range(tr.R)}
    first = True
    for r in window_order(tr.R, tr.rank):
        handles[r].wait()
        if hi > lo and r * w < l:
            ctx.shard_ks_window(kind, step, D_all[r, :cnt], r, w, a, lo, l, first)
            first = False
    if hi > lo:
        ctx.shard_ks_combine(kind, step, a, lo, l, out)
    return out


def sharded_rescale(ctx, tr: Transport, ct, L: int, l: int, count: int, out_alloc):
    """Sharded RESCALE (Eq. 1): the owner of limb l-1 produces its coefficient form X,
    broadcasts it, and every rank floors its own limbs < l-1."""
    lo, hi, w = limb_shard(L, tr.R, tr.rank, l)
    owner = (l - 1) // w
    X = torch.empty((count, 2, ctx.N), dtype=torch.int64, device=ctx.device)
    if tr.rank == owner:
        ctx.shard_rescale_last(ct, lo, l, X)
    tr.broadcast(X, owner)
    hi2 = min(hi, l - 1)
    if hi2 <= lo:
        return None
    out = out_alloc(count, hi2 - lo)
    return ctx.shard_rescale_apply(X, ct, lo, l, out)
