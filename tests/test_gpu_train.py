"""GPU parity of the encrypted training step: gradient sums and the
updated model are bit-exact with the oracle composer on identical imported inputs; the
decrypted update matches the float64 minibatch gradient step."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1908_06972_b200 import synth  # noqa: E402


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).cuda()


def _host(t):
    return t.cpu().numpy().view(np.uint64)


# (log_n, limb bits, special bits, alpha, K, scale, decode tolerance): the per-limb key switching of
# reading A6, and the hybrid key switching the bench trains with (FP64-mode 41-bit special primes:
# fused ModUp row phase + inner product, fused ModDown + rescale tail) on an all-FP64 chain
TRAIN_CFGS = [(10, [60] + [40] * 10, 60, 1, 1, 2.0 ** 40, 1e-4),
              (12, [41] + [30] * 10, 41, 4, 4, 2.0 ** 30, 1e-2),
              (12, [40] + [30] * 10, 40, 4, 4, 2.0 ** 30, 1e-2)]


@pytest.mark.parametrize("cfg", TRAIN_CFGS, ids=["alpha1", "hybrid_f64", "hybrid_compact_keys"])
def test_train_step_bit_exact(oracle_mod, cfg):
    from paper_1908_06972_b200 import ckks
    log_n, bits, sp_bits, alpha, K, scale, tol = cfg
    m, n, c, E, eta = 300, 3, 2, 3, 0.5
    p = oracle_mod.toy_params(log_n, bits, sp_bits, scale=scale, alpha=alpha, n_special=K)
    ctx = ckks.Context(log_n, bits, sp_bits, scale, n_special=K, digit_limbs=alpha)
    assert ctx.q == p.q and ctx.special == p.special
    t = p.slots
    kr = synth.KeyRandomness(3, p.log_n, p.q, p.P)
    pk = oracle_mod.keygen_public(p, kr.s, kr.pk_a, kr.pk_e)
    rlk = oracle_mod.keygen_relin(p, kr.s, *kr.switch_key(0, dnum=p.dnum, special=p.special))
    ctx.import_switch_key(0, 0, _cuda(rlk))
    gk = {}
    for i in range(log_n - 1):
        kappa, key = oracle_mod.keygen_galois(p, kr.s, 1 << i, *kr.switch_key(1 + i, dnum=p.dnum, special=p.special))
        gk[kappa] = key
        ctx.import_switch_key(1, 1 << i, _cuda(key))
    g = synth.rng(3)
    H = g.uniform(-1, 1, (m, n))
    O = g.uniform(-1, 1, (n, c))
    enc = lambda z, tag: oracle_mod.encrypt(p, pk, oracle_mod.encode(p, z), *kr.enc(tag))
    Hc = [enc(np.pad(H[:, j], (0, t - m)), 100 + j) for j in range(n)]
    Oc = [enc(np.pad(O[j], (0, t - c)), 200 + j) for j in range(n)]
    exs, plain = [], []
    for k in range(E):
        v, w = synth.bag(synth.rng(50 + k), m, 40)
        exs.append((enc(np.pad(v, (0, t - m)), 300 + k), w, k % c))
        plain.append((v, w, k % c))
    negs, mask = oracle_mod.train_plaintexts(p, Hc, Oc, exs, c)
    GH, GO = oracle_mod.train_gradients(p, Hc, Oc, exs, c, rlk, gk, (negs, mask))
    Hn, On = oracle_mod.train_update(p, Hc, Oc, GH, GO, eta)

    imp = lambda cts, scale: ctx.import_coeffs(_cuda(np.stack([np.stack(x.c) for x in cts])), p.L, scale)
    Hd, Od, Bd = imp(Hc, Hc[0].scale), imp(Oc, Oc[0].scale), imp([x[0] for x in exs], exs[0][0].scale)
    gs, gl = ctx.privft_train_plan(Hd, Od, Bd)
    assert gs == negs[0].scale and gl == negs[0].level
    NEG = ctx.import_coeffs(_cuda(np.stack([x.m for x in negs])[:, None]), gl, gs)
    MK = ctx.import_coeffs(_cuda(mask.m[None, None]), gl, mask.scale)
    gH, gO = ctx.privft_train_grad(Hd, Od, Bd, [x[1] for x in exs], [x[2] for x in exs], c, NEG, MK)
    assert gH.level == GH[0].level and gO.level == GO[0].level and gH.scale == GH[0].scale
    got = _host(ctx.export_coeffs(gH))
    for j in range(n):
        assert np.array_equal(got[j, 0], GH[j].c[0]) and np.array_equal(got[j, 1], GH[j].c[1]), j
    got = _host(ctx.export_coeffs(gO))
    for j in range(n):
        assert np.array_equal(got[j, 0], GO[j].c[0]) and np.array_equal(got[j, 1], GO[j].c[1]), j
    Hn_d, On_d = ctx.privft_train_update(Hd, Od, gH, gO, eta)
    gh_, go_ = _host(ctx.export_coeffs(Hn_d)), _host(ctx.export_coeffs(On_d))
    for j in range(n):
        assert np.array_equal(gh_[j, 0], Hn[j].c[0]) and np.array_equal(gh_[j, 1], Hn[j].c[1]), j
        assert np.array_equal(go_[j, 0], On[j].c[0]) and np.array_equal(go_[j, 1], On[j].c[1]), j
    Hw, Ow = oracle_mod.train_plain(H, O, plain, c, eta)
    dec = lambda ct: oracle_mod.decode(p, oracle_mod.decrypt(p, kr.s, ct)).real
    for j in range(n):
        assert np.max(np.abs(dec(Hn[j])[:m] - Hw[:, j])) < tol
        assert np.max(np.abs(dec(On[j])[:c] - Ow[j])) < tol
