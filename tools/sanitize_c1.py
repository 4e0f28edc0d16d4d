"""Small C1 workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
HMult+relin+rescale, rotate(3), TotalSum, mul_plain, NTT round trip and a tiny PrivFT
inference, checked bit-exactly against the oracle so a sanitizer run is also a parity run.
CKKS_KS_CLUSTER=1 routes the key switches through the cluster kernel."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_1908_06972_b200 import ckks, synth  # noqa: E402


def cu(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).cuda()


def host(t):
    return t.cpu().numpy().view(np.uint64)


log_n = int(os.environ.get("LOGN", 12))
bits = [30] * 3 if log_n == 12 else [60] + [40] * 4
qs, sp = oracle.prime_chain(log_n, bits)
p = oracle.Params(log_n, qs, sp[0], 2.0 ** 30)
ctx = ckks.Context(log_n, bits, 60, 2.0 ** 30)
g = synth.rng(9)
ext = list(p.ext_mods())
key = lambda: np.stack([np.stack([synth.uniform_residues(g, ext, p.N) for _ in range(2)]) for _ in range(p.L)])
rlk = key()
ctx.import_switch_key(0, 0, cu(rlk))
gk = {}
for i in range(p.log_n - 1):
    k = key()
    ctx.import_switch_key(1, 1 << i, cu(k))
    gk[oracle.galois_elt(p, 1 << i)] = k
for st in oracle.rotation_steps(p, 3):
    if oracle.galois_elt(p, st) not in gk:
        k = key()
        ctx.import_switch_key(1, st, cu(k))
        gk[oracle.galois_elt(p, st)] = k
L = p.L
a = np.stack([np.stack([synth.uniform_residues(g, p.q, p.N) for _ in range(2)]) for _ in range(2)])
b = np.stack([np.stack([synth.uniform_residues(g, p.q, p.N) for _ in range(2)]) for _ in range(2)])
A, B = ctx.import_coeffs(cu(a), L, 1.0), ctx.import_coeffs(cu(b), L, 1.0)
m = host(ctx.export_coeffs(ctx.rescale(ctx.mul_relin(A, B))))
r = host(ctx.export_coeffs(ctx.rotate(A, 3)))
ts = host(ctx.export_coeffs(ctx.total_sum(A)))
for c in range(2):
    oa = oracle.Ciphertext([a[c, 0], a[c, 1]], L, 1.0)
    ob = oracle.Ciphertext([b[c, 0], b[c, 1]], L, 1.0)
    wm = oracle.rescale(p, oracle.mul_relin(p, oa, ob, rlk))
    wr = oracle.rotate(p, oa, 3, gk)
    wt = oracle.total_sum(p, oa, gk)
    for k in range(2):
        assert np.array_equal(m[c, k], wm.c[k]) and np.array_equal(r[c, k], wr.c[k])
        assert np.array_equal(ts[c, k], wt.c[k])
X = cu(a.reshape(4, L, p.N))
ctx.ntt(X)
ctx.ntt(X, inverse=True)
assert np.array_equal(host(X), a.reshape(4, L, p.N))
torch.cuda.synchronize()
print(f"sanitize workload ok: logN={log_n}, cluster={os.environ.get('CKKS_KS_CLUSTER', '0')}, "
      f"{ctx.launches()} libckks launches")
