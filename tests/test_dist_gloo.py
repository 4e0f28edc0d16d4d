"""World-size-2 gloo tests of the multi-GPU host logic on CPU: query
sharding and the all-gather layout feeding the modular add.  The modular reduction here
is the oracle's poly_add (test-only); on GPU it is ckks_modadd_gathered."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1908_06972_b200.dist import shard_range


def test_shard_range_partitions():
    for total in (0, 1, 7, 64, 100):
        for world in (1, 2, 3, 8):
            spans = [shard_range(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, out):
    import torch
    import torch.distributed as dist

    from paper_1908_06972_b200 import synth
    from paper_1908_06972_b200.dist import gather_limbs
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = synth.rng(100 + rank)
    local = np.stack([np.stack([synth.uniform_residues(g, q, 16) for _ in range(2)]) for _ in range(3)])
    t = torch.from_numpy(local.view(np.int64).copy())
    gathered = gather_limbs(t)
    out[rank] = gathered.numpy().view(np.uint64).copy()
    dist.destroy_process_group()


def test_gather_layout_and_modular_sum(oracle_mod):
    q = oracle_mod.prime_scan(3, 40, 0, 3)
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), q, out), nprocs=world, join=True)
    from paper_1908_06972_b200 import synth
    parts = []
    for r in range(world):
        g = synth.rng(100 + r)
        parts.append(np.stack([np.stack([synth.uniform_residues(g, q, 16) for _ in range(2)]) for _ in range(3)]))
    for r in range(world):
        got = out[r]
        assert got.shape == (world, 3, 2, 3, 16)
        for rr in range(world):  # gathered[rr] is rank rr's bit-identical buffer
            assert np.array_equal(got[rr], parts[rr])
        # modular sum over the gathered axis (oracle reduction == what ckks_modadd_gathered computes)
        s = got[0]
        for rr in range(1, world):
            s = np.stack([np.stack([oracle_mod.poly_add(s[c, k], got[rr][c, k], q, 4) for k in range(2)])
                          for c in range(3)])
        want = np.stack([np.stack([oracle_mod.poly_add(parts[0][c, k], parts[1][c, k], q, 4) for k in range(2)])
                         for c in range(3)])
        assert np.array_equal(s, want)
