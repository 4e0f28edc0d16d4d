"""One rank of the f3 peer-memory modular all-reduce test (launched by test_gpu_p2p.py as
R processes; all may share one GPU -- CUDA IPC maps another process's allocation on the
same device just as on a peer).  Prints one JSON line: this rank's result digest."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1908_06972_b200 import ckks, synth  # noqa: E402
from paper_1908_06972_b200.dist import PeerModSum  # noqa: E402


def rank_input(q, N, count, level, cap, rank):
    """Seeded residues [count][2][cap][N] (limbs >= level are left as a sentinel)."""
    g = synth.rng(5000 + rank)
    x = np.full((count, 2, cap, N), 0xDEAD, dtype=np.uint64)
    for c in range(count):
        for k in range(2):
            x[c, k, :level] = synth.uniform_residues(g, q[:level], N)
    return x


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dev = int(os.environ.get("P2P_DEVICE", "0"))
    torch.cuda.set_device(dev)
    count, level, cap = 3, 3, 4
    ctx = ckks.Context(12, [30, 30, 30, 30], 60, 2.0 ** 30, device=dev)
    x = rank_input(ctx.q, ctx.N, count, level, cap, rank)
    t = torch.from_numpy(x.view(np.int64)).cuda(dev)
    buf = ckks.Buf(t, level, 1.0)
    op = PeerModSum(ctx, buf)
    op()
    got_inplace = t.cpu().numpy().view(np.uint64).copy()
    # second form: separate outputs, explicit pointer lists
    t2 = torch.from_numpy(rank_input(ctx.q, ctx.N, count, level, cap, rank).view(np.int64)).cuda(dev)
    o2 = torch.zeros_like(t2)
    hs = [None] * world
    dist.all_gather_object(hs, (ctx.ipc_export(t2), ctx.ipc_export(o2)))
    ins, outs = [], []
    for r, ((hi, oi), (ho, oo)) in enumerate(hs):
        ins.append(t2.data_ptr() if r == rank else ctx.ipc_open(hi, oi))
        outs.append(o2.data_ptr() if r == rank else ctx.ipc_open(ho, oo))
    torch.cuda.synchronize()
    dist.barrier()
    ctx.p2p_modsum(ins, outs, rank, ckks.Buf(t2, level, 1.0))
    torch.cuda.synchronize()
    dist.barrier()
    got_sep = o2.cpu().numpy().view(np.uint64).copy()
    src_kept = np.array_equal(t2.cpu().numpy().view(np.uint64), rank_input(ctx.q, ctx.N, count, level, cap, rank))
    for r in range(world):
        if r != rank:
            ctx.ipc_close(ins[r])
            ctx.ipc_close(outs[r])
    op.close()
    dist.barrier()
    np.save(os.path.join(os.environ["P2P_OUT"], f"rank{rank}_inplace.npy"), got_inplace)
    np.save(os.path.join(os.environ["P2P_OUT"], f"rank{rank}_sep.npy"), got_sep)
    print(json.dumps({"rank": rank, "src_kept": bool(src_kept), "q": ctx.q}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
