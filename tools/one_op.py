"""Set up a context like tools/time_ops.py and run one op `calls` times (for ncu captures
filtered with --nvtx --nvtx-include "<op>/"):
python tools/one_op.py log_n L op [calls] [count] [alpha] [K] [special bits]
op: hmult (mul_relin_rescale) | rotate | ntt"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import gaussian, uniform_limbs  # noqa: E402
from paper_1908_06972_b200 import ckks  # noqa: E402

log_n, L, op = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
calls = int(sys.argv[4]) if len(sys.argv) > 4 else 2
count = int(sys.argv[5]) if len(sys.argv) > 5 else 1
alpha = int(sys.argv[6]) if len(sys.argv) > 6 else 1
K = int(sys.argv[7]) if len(sys.argv) > 7 else 1
sp_bits = int(sys.argv[8]) if len(sys.argv) > 8 else 60
dev = torch.device("cuda", 0)
gen = torch.Generator(device=dev)
gen.manual_seed(1)
bits = [40] * L if log_n >= 14 else [60] + [40] * (L - 1)
ctx = ckks.Context(log_n, bits, sp_bits, 2.0 ** 40, n_special=K, digit_limbs=alpha)
N = ctx.N
ctx.set_secret(torch.randint(0, 2, (N,), dtype=torch.int64, device=dev, generator=gen))
ext = ctx.q + ctx.special
D = ctx.dnum
ctx.keygen_relin(uniform_limbs(torch, (D,), ext, N, dev, gen), gaussian(torch, (D, N), dev, gen))
ctx.keygen_galois(1, uniform_limbs(torch, (D,), ext, N, dev, gen), gaussian(torch, (D, N), dev, gen))
A = ckks.Buf(uniform_limbs(torch, (count, 2), ctx.q, N, dev, gen), L, ctx.scale)
B = ckks.Buf(uniform_limbs(torch, (count, 2), ctx.q, N, dev, gen), L, ctx.scale)
T = ctx.alloc(count, 2, L)
R = ctx.alloc(count, 2, L)
torch.cuda.synchronize()
for _ in range(calls):
    if op == "hmult":
        ctx.mul_relin_rescale(A, B, out=T)
    elif op == "rotate":
        ctx.rotate(A, 1, out=R)
    torch.cuda.synchronize()
print("done")
