"""Limb-sharded key switching on ONE GPU with R logical shards: the
all-gather is emulated by stacking the shards' digit buffers.  The sharded HMult+relin+
rescale and rotation must be bit-identical to the unsharded op (and to the oracle)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1908_06972_b200 import synth  # noqa: E402
from paper_1908_06972_b200.dist import limb_shard, window_order  # noqa: E402


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).cuda()


def _host(t):
    return t.cpu().numpy().view(np.uint64)


def run_sharded(ctx, kind, step, a_full, b_full, L, l, R, pipelined=False):
    """Emulate R ranks on one device; returns the assembled (un-sharded) result coefficients
    after the key switch and (kind 0) the rescale."""
    from paper_1908_06972_b200 import ckks
    cnt, N = a_full.count, ctx.N
    shards = []
    for r in range(R):
        lo, hi, w = limb_shard(L, R, r, l)
        if hi <= lo:
            shards.append(None)
            continue
        a = ckks.Buf(a_full.t[:, :, lo:hi].contiguous(), hi - lo, a_full.scale)
        b = ckks.Buf(b_full.t[:, :, lo:hi].contiguous(), hi - lo, b_full.scale) if b_full is not None else None
        shards.append((lo, hi, a, b))
    w = limb_shard(L, R, 0, l)[2]
    outs, D = [], torch.zeros((R, cnt, w, N), dtype=torch.int64, device="cuda")
    for r, sh in enumerate(shards):
        if sh is None:
            outs.append(None)
            continue
        lo, hi, a, b = sh
        out = ctx.alloc(cnt, 2, hi - lo)
        ctx.shard_ks_digits(kind, step, a, b, lo, l, w, out, D[r])
        outs.append(out)
    for r, sh in enumerate(shards):  # "after the all-gather": every rank sees D
        if sh is None:
            continue
        lo, hi, a, b = sh
        if pipelined:  # row f3: the digit windows folded in one by one (own first), then ModDown
            first = True
            for rr in window_order(R, r):
                if rr * w < l:
                    ctx.shard_ks_window(kind, step, D[rr], rr, w, a, lo, l, first)
                    first = False
            ctx.shard_ks_combine(kind, step, a, lo, l, outs[r])
        else:
            ctx.shard_ks_finish(kind, step, D, R, w, a, lo, l, outs[r])
    if kind == 1:
        return torch.cat([o.t for o in outs if o is not None], dim=2), outs[0].scale
    owner = (l - 1) // w
    lo_o = shards[owner][0]
    X = torch.empty((cnt, 2, N), dtype=torch.int64, device="cuda")
    ctx.shard_rescale_last(outs[owner], lo_o, l, X)
    res = []
    for r, sh in enumerate(shards):
        if sh is None:
            continue
        lo, hi, a, b = sh
        if min(hi, l - 1) > lo:
            o = ctx.alloc(cnt, 2, min(hi, l - 1) - lo)
            ctx.shard_rescale_apply(X, outs[r], lo, l, o)
            res.append(o)
    return torch.cat([o.t for o in res], dim=2), res[0].scale


@pytest.mark.parametrize("pipelined", [False, True])
@pytest.mark.parametrize("R", [2, 3])
def test_sharded_matches_oracle_c1(oracle_mod, R, pipelined):
    from paper_1908_06972_b200 import ckks
    p = oracle_mod.preset("C1")
    ctx = ckks.Context(p.log_n, [30] * 3, 60, p.scale)
    kr = synth.KeyRandomness(1, p.log_n, p.q, p.P)
    rlk = oracle_mod.keygen_relin(p, kr.s, *kr.switch_key(0))
    kappa, gk = oracle_mod.keygen_galois(p, kr.s, 1, *kr.switch_key(101))
    ctx.import_switch_key(0, 0, _cuda(rlk))
    ctx.import_switch_key(1, 1, _cuda(gk))
    g = synth.rng(5)
    a = np.stack([np.stack([synth.uniform_residues(g, p.q, p.N) for _ in range(2)]) for _ in range(2)])
    b = np.stack([np.stack([synth.uniform_residues(g, p.q, p.N) for _ in range(2)]) for _ in range(2)])
    A, B = ctx.import_coeffs(_cuda(a), 3, 1.0), ctx.import_coeffs(_cuda(b), 3, 1.0)
    got, scale = run_sharded(ctx, 0, 0, A, B, 3, 3, R, pipelined)
    got = _host(ctx.export_coeffs(ckks.Buf(got.contiguous(), 2, scale)))
    rot, _ = run_sharded(ctx, 1, 1, A, None, 3, 3, R, pipelined)
    rot = _host(ctx.export_coeffs(ckks.Buf(rot.contiguous(), 3, 1.0)))
    for c in range(2):
        oa = oracle_mod.Ciphertext([a[c, 0], a[c, 1]], 3, 1.0)
        ob = oracle_mod.Ciphertext([b[c, 0], b[c, 1]], 3, 1.0)
        want = oracle_mod.rescale(p, oracle_mod.mul_relin(p, oa, ob, rlk))
        wr = oracle_mod.apply_galois(p, oa, kappa, gk)
        for k in range(2):
            assert np.array_equal(got[c, k], want.c[k]), (c, k)
            assert np.array_equal(rot[c, k], wr.c[k]), (c, k)


@pytest.mark.parametrize("pipelined", [False, True])
@pytest.mark.parametrize("R", [2, 3, 8])
def test_sharded_bit_identical_to_unsharded_c2(R, pipelined):
    """N = 2^14, L = 8, 3 ciphertexts: R logical shards vs the single-GPU op."""
    from paper_1908_06972_b200 import ckks
    ctx = ckks.Context(14, [40] * 8, 60, 2.0 ** 40)
    dev = torch.device("cuda")
    gen = torch.Generator(device=dev)
    gen.manual_seed(3)
    N, L = ctx.N, 8

    def uni(prefix, primes):
        t = torch.empty((*prefix, len(primes), N), dtype=torch.int64, device=dev)
        for i, q in enumerate(primes):
            t[..., i, :] = torch.randint(0, q, (*prefix, N), dtype=torch.int64, device=dev, generator=gen)
        return t

    ctx.set_secret(torch.randint(0, 2, (N,), dtype=torch.int64, device=dev, generator=gen))
    ext = ctx.q + [ctx.P]
    e = lambda: torch.randint(-5, 6, (L, N), dtype=torch.int64, device=dev, generator=gen)
    ctx.keygen_relin(uni((L,), ext), e())
    ctx.keygen_galois(-4, uni((L,), ext), e())
    for l in (8, 5):
        A = ckks.Buf(uni((3, 2), ctx.q[:l]).contiguous(), l, 1.0)
        B = ckks.Buf(uni((3, 2), ctx.q[:l]).contiguous(), l, 1.0)
        want = ctx.rescale(ctx.mul_relin(A, B))
        got, _ = run_sharded(ctx, 0, 0, A, B, L, l, R, pipelined)
        assert torch.equal(got, want.t[:, :, :l - 1])
        want_r = ctx.rotate(A, -4)
        got_r, _ = run_sharded(ctx, 1, -4, A, None, L, l, R, pipelined)
        assert torch.equal(got_r, want_r.t[:, :, :l])
