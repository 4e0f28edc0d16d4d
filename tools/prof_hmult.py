"""Run a few C3 HMult+relin+rescale ops (for ncu captures): python tools/prof_hmult.py [iters] [log_n] [L]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import gaussian, uniform_limbs  # noqa: E402
from paper_1908_06972_b200 import ckks  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 3
log_n = int(sys.argv[2]) if len(sys.argv) > 2 else 16
L = int(sys.argv[3]) if len(sys.argv) > 3 else 30
dev = torch.device("cuda", 0)
gen = torch.Generator(device=dev)
gen.manual_seed(1)
ctx = ckks.Context(log_n, [40] * L, 60, 2.0 ** 40)
N = ctx.N
ctx.set_secret(torch.randint(0, 2, (N,), dtype=torch.int64, device=dev, generator=gen))
ext = ctx.q + [ctx.P]
ctx.keygen_relin(uniform_limbs(torch, (L,), ext, N, dev, gen), gaussian(torch, (L, N), dev, gen))
A = ckks.Buf(uniform_limbs(torch, (1, 2), ctx.q, N, dev, gen), L, ctx.scale)
B = ckks.Buf(uniform_limbs(torch, (1, 2), ctx.q, N, dev, gen), L, ctx.scale)
T = ctx.alloc(1, 2, L)
O = ctx.alloc(1, 2, L - 1)
for _ in range(iters):
    ctx.rescale(ctx.mul_relin(A, B, out=T), out=O)
torch.cuda.synchronize()
print("done")
