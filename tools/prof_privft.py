"""A few PrivFT inference steps with bench.py's exact setup (for ncu captures):
python tools/prof_privft.py [batch] [steps] [n]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1908_06972_b200 import ckks  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 32
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
n = int(sys.argv[3]) if len(sys.argv) > 3 else 300
dev = torch.device("cuda", 0)
gen = torch.Generator(device=dev)
gen.manual_seed(1234)
C4 = bench.C4
ctx = ckks.Context(C4["log_n"], C4["limb_bits"], C4["special_bits"], C4["scale"])
N, L = ctx.N, ctx.L
K = -(-500000 // (N // 2))
bench.setup_keys(torch, ctx, [1 << i for i in range(ctx.log_n - 1)], gen)
Hp = ckks.Buf(bench.uniform_limbs(torch, (n * K, 1), ctx.q, N, dev, gen), L, ctx.scale)
Op = ckks.Buf(bench.uniform_limbs(torch, (n, 1), ctx.q[:L - 2], N, dev, gen), L - 2, ctx.scale)
model = ctx.privft_model_wrap(Hp, Op, 500000, n, 4)
bag = ckks.Buf(bench.uniform_limbs(torch, (B * K, 2), ctx.q, N, dev, gen), L, ctx.scale)
w = [100 + i for i in range(B)]
scores = ctx.alloc(B, 2, L - 4, L - 3)
for _ in range(steps):
    ctx.privft_infer(model, bag, w, True, out=scores)
torch.cuda.synchronize()
print("done")

if "--table" in sys.argv:
    peaks = bench.int_peak()
    ctx.profile(True)
    for _ in range(steps):
        ctx.privft_infer(model, bag, w, True, out=scores)
    torch.cuda.synchronize()
    ctx.profile(False)
    prof = ctx.profile_read()
    tot = sum(v["ms"] for v in prof.values())
    print(f"{'kernel':22s} {'ms/step':>9s} {'share':>6s} {'Gbfly/s':>9s} {'alu frac':>8s} {'GB/s':>8s} launches/step")
    for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"]):
        sec = v["ms"] * 1e-3
        eq = bench.bfly_equiv(v, peaks)
        print(f"{k:22s} {v['ms'] / steps:9.2f} {v['ms'] / tot:6.3f} {eq / sec / 1e9:9.1f} "
              f"{eq / sec / peaks['bfly_per_s']:8.3f} {v['bytes'] / sec / 1e9:8.0f} {v['launches'] // steps}")
