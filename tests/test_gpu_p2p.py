"""GPU parity of the fused peer-memory modular all-reduce.

R worker processes (tests/p2p_worker.py, gloo rendezvous on 127.0.0.1) map each other's
buffers through CUDA IPC and run ckks_p2p_modsum; every rank must end with the limb-wise
sum of all ranks' inputs mod q_i, computed here with the oracle's poly_add.  Limbs past
`level` (capacity padding) must be untouched; separate-output form must leave inputs intact.
R = 3 and 4 give uneven slices of the 18 limb rows."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("R", [2, 3, 4])
def test_p2p_modsum_matches_oracle(oracle_mod, tmp_path, R):
    sys.path.insert(0, HERE)
    import p2p_worker
    port = _free_port()
    procs = []
    for r in range(R):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(R), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                   P2P_OUT=str(tmp_path))
        procs.append(subprocess.Popen([sys.executable, os.path.join(HERE, "p2p_worker.py")], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
    outs = []
    for p in procs:
        o, e = p.communicate(timeout=300)
        assert p.returncode == 0, e[-3000:]
        outs.append(json.loads(o.strip().splitlines()[-1]))
    q = outs[0]["q"]
    count, level, cap, N = 3, 3, 4, 1 << 12
    xs = [p2p_worker.rank_input(q, N, count, level, cap, r) for r in range(R)]
    want = xs[0].copy()
    for c in range(count):
        for k in range(2):
            acc = xs[0][c, k, :level]
            for r in range(1, R):
                acc = oracle_mod.poly_add(acc, xs[r][c, k, :level], q[:level], 12)
            want[c, k, :level] = acc
    for r in range(R):
        assert outs[r]["src_kept"]
        got = np.load(tmp_path / f"rank{r}_inplace.npy")
        assert np.array_equal(got, want), r  # includes the untouched padding limb
        sep = np.load(tmp_path / f"rank{r}_sep.npy")
        assert np.array_equal(sep[:, :, :level], want[:, :, :level]), r
        assert not np.any(sep[:, :, level:]), r
