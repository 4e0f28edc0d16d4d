"""Time HMult+relin+rescale / rotate at a config with CUDA events; prints per-kernel split.
python tools/time_ops.py [log_n] [L] [iters] [count]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import gaussian, uniform_limbs  # noqa: E402
from paper_1908_06972_b200 import ckks  # noqa: E402

log_n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
L = int(sys.argv[2]) if len(sys.argv) > 2 else 30
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 10
count = int(sys.argv[4]) if len(sys.argv) > 4 else 1
alpha = int(sys.argv[5]) if len(sys.argv) > 5 else 1
K = int(sys.argv[6]) if len(sys.argv) > 6 else 1
sp_bits = int(sys.argv[7]) if len(sys.argv) > 7 else 60
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
O = ctx.alloc(count, 2, L - 1)
R = ctx.alloc(count, 2, L)


def timeit(f, prof=False):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    if prof:
        ctx.profile(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        f()
    e1.record()
    torch.cuda.synchronize()
    if prof:
        ctx.profile(False)
        return e0.elapsed_time(e1) * 1e3 / iters, ctx.profile_read()
    return e0.elapsed_time(e1) * 1e3 / iters, None


hm0 = lambda: ctx.rescale(ctx.mul_relin(A, B, out=T), out=O)
hm = lambda: ctx.mul_relin_rescale(A, B, out=T)
rot = lambda: ctx.rotate(A, 1, out=R)
tag = f"logN={log_n} L={L} alpha={alpha} K={K}x{sp_bits}b count={count}"
us, _ = timeit(hm0)
print(f"{tag}: HMult+relin, rescale {us:.1f} us/batch ({us / count:.2f} us/ct) [two calls]")
us, _ = timeit(hm)
print(f"{tag}: HMult+relin+rescale {us:.1f} us/batch ({us / count:.2f} us/ct) [fused]")
us, _ = timeit(rot)
print(f"{tag}: rotate(1)          {us:.1f} us/batch ({us / count:.2f} us/ct)")
us, prof = timeit(hm, prof=True)
tot = sum(v["ms"] for v in prof.values())
print("   profiled HMult", " ".join(f"{k}={v['ms'] * 1e3 / iters:.1f}us" for k, v in
                                    sorted(prof.items(), key=lambda kv: -kv[1]["ms"])))
