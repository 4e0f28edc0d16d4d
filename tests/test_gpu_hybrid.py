"""GPU parity of hybrid key switching (alpha-limb digits, K special
primes, fast base conversion) against the oracle: mul_relin, rescale and rotation
bit-exact at full and partial-digit levels; library keygen == oracle keygen."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1908_06972_b200 import synth  # noqa: E402


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).cuda()


def _host(t):
    return t.cpu().numpy().view(np.uint64)


@pytest.fixture(scope="module", params=[(2, 2), (3, 2), (4, 3)])
def world(request, oracle_mod):
    from paper_1908_06972_b200 import ckks
    alpha, K = request.param
    p = oracle_mod.toy_params(12, [30] * 6, 60, alpha=alpha, n_special=K)
    ctx = ckks.Context(12, [30] * 6, 60, 2.0 ** 20, n_special=K, digit_limbs=alpha)
    assert ctx.q == p.q and ctx.special == p.special
    kr = synth.KeyRandomness(4, p.log_n, p.q, p.P)
    ar, er = kr.switch_key(0, dnum=p.dnum, special=p.special)
    rlk = oracle_mod.keygen_relin(p, kr.s, ar, er)
    kappa, gk = oracle_mod.keygen_galois(p, kr.s, 1, *kr.switch_key(7, dnum=p.dnum, special=p.special))
    ctx.import_switch_key(0, 0, _cuda(rlk))
    ctx.import_switch_key(1, 1, _cuda(gk))
    return dict(p=p, ctx=ctx, kr=kr, rlk=rlk, gk={kappa: gk}, kappa=kappa, ar=ar, er=er)


def rand_ct(p, count, level, seed):
    g = synth.rng(seed)
    return np.stack([np.stack([synth.uniform_residues(g, p.q[:level], p.N) for _ in range(2)])
                     for _ in range(count)])


@pytest.mark.parametrize("level", [6, 5, 3, 2])
def test_hybrid_mul_relin_rescale_bit_exact(oracle_mod, world, level):
    p, ctx = world["p"], world["ctx"]
    a, b = rand_ct(p, 2, level, 10), rand_ct(p, 2, level, 11)
    A, B = ctx.import_coeffs(_cuda(a), level, 1.0), ctx.import_coeffs(_cuda(b), level, 1.0)
    M = ctx.mul_relin(A, B)
    got = _host(ctx.export_coeffs(M))
    got_r = _host(ctx.export_coeffs(ctx.rescale(M)))
    got_f = _host(ctx.export_coeffs(ctx.mul_relin_rescale(A, B)))  # fused ModDown + rescale tail
    for c in range(2):
        oa = oracle_mod.Ciphertext([a[c, 0], a[c, 1]], level, 1.0)
        ob = oracle_mod.Ciphertext([b[c, 0], b[c, 1]], level, 1.0)
        want = oracle_mod.mul_relin(p, oa, ob, world["rlk"])
        wr = oracle_mod.rescale(p, want)
        for k in range(2):
            assert np.array_equal(got[c, k], want.c[k]), (c, k)
            assert np.array_equal(got_r[c, k], wr.c[k]), (c, k)
            assert np.array_equal(got_f[c, k], wr.c[k]), (c, k)


@pytest.mark.parametrize("level", [6, 4])
def test_hybrid_rotate_bit_exact(oracle_mod, world, level):
    p, ctx = world["p"], world["ctx"]
    a = rand_ct(p, 2, level, 20)
    A = ctx.import_coeffs(_cuda(a), level, 1.0)
    got = _host(ctx.export_coeffs(ctx.rotate(A, 1)))
    for c in range(2):
        want = oracle_mod.apply_galois(p, oracle_mod.Ciphertext([a[c, 0], a[c, 1]], level, 1.0), world["kappa"],
                                       world["gk"][world["kappa"]])
        assert np.array_equal(got[c, 0], want.c[0]) and np.array_equal(got[c, 1], want.c[1])


def test_hybrid_keygen_matches_oracle(oracle_mod, world):
    from paper_1908_06972_b200 import ckks
    p, kr = world["p"], world["kr"]
    ctx = ckks.Context(12, [30] * 6, 60, 2.0 ** 20, n_special=p.K, digit_limbs=p.alpha)
    ctx.set_secret(_cuda(kr.s))
    ctx.keygen_relin(_cuda(world["ar"]), _cuda(world["er"]))
    a, b = rand_ct(p, 1, 6, 30), rand_ct(p, 1, 6, 31)
    A, B = ctx.import_coeffs(_cuda(a), 6, 1.0), ctx.import_coeffs(_cuda(b), 6, 1.0)
    got = _host(ctx.export_coeffs(ctx.mul_relin(A, B)))
    want = oracle_mod.mul_relin(p, oracle_mod.Ciphertext([a[0, 0], a[0, 1]], 6, 1.0),
                                oracle_mod.Ciphertext([b[0, 0], b[0, 1]], 6, 1.0), world["rlk"])
    assert np.array_equal(got[0, 0], want.c[0]) and np.array_equal(got[0, 1], want.c[1])


@pytest.mark.parametrize("bits,alpha,K", [([30] * 20, 10, 7), ([40] * 12, 5, 4)])
@pytest.mark.parametrize("conv_v1", [False, True])
def test_hybrid_wide_digits_bit_exact(oracle_mod, monkeypatch, bits, alpha, K, conv_v1):
    """The bench's digit shape (alpha = 10, K = 7: alpha-specialised conversion kernels, FP64
    accumulation for the 30/40-bit slots, 128-bit for the 60-bit special slots) and a
    partial last digit (12 = 2 x 5 + 2), with the v2 and v1 conversion kernels."""
    from paper_1908_06972_b200 import ckks
    if conv_v1:
        monkeypatch.setenv("CKKS_MODUP_CONV", "1")
        monkeypatch.setenv("CKKS_MODDOWN_CONV", "1")
    L = len(bits)
    p = oracle_mod.toy_params(12, bits, 60, alpha=alpha, n_special=K)
    ctx = ckks.Context(12, bits, 60, 2.0 ** 20, n_special=K, digit_limbs=alpha)
    assert ctx.q == p.q and ctx.special == p.special
    kr = synth.KeyRandomness(9, p.log_n, p.q, p.P)
    rlk = oracle_mod.keygen_relin(p, kr.s, *kr.switch_key(0, dnum=p.dnum, special=p.special))
    ctx.import_switch_key(0, 0, _cuda(rlk))
    for level in (L, L - 3):
        a, b = rand_ct(p, 2, level, 40 + level), rand_ct(p, 2, level, 50 + level)
        A, B = ctx.import_coeffs(_cuda(a), level, 1.0), ctx.import_coeffs(_cuda(b), level, 1.0)
        got = _host(ctx.export_coeffs(ctx.mul_relin(A, B)))
        got_f = _host(ctx.export_coeffs(ctx.mul_relin_rescale(A, B)))
        for c in range(2):
            want = oracle_mod.mul_relin(p, oracle_mod.Ciphertext([a[c, 0], a[c, 1]], level, 1.0),
                                        oracle_mod.Ciphertext([b[c, 0], b[c, 1]], level, 1.0), rlk)
            assert np.array_equal(got[c, 0], want.c[0]) and np.array_equal(got[c, 1], want.c[1]), (level, c)
            wr = oracle_mod.rescale(p, want)
            assert np.array_equal(got_f[c, 0], wr.c[0]) and np.array_equal(got_f[c, 1], wr.c[1]), (level, c)
    ctx.close()


@pytest.mark.parametrize("L,alpha,K,sp_bits,variant", [(12, 4, 4, 41, ""), (20, 10, 10, 41, ""), (9, 3, 3, 41, ""),
                                                         (20, 10, 10, 40, ""), (12, 4, 4, 40, ""),
                                                         (20, 10, 10, 40, "CKKS_HYB_FUSED_IP=0"),
                                                         (20, 10, 10, 40, "CKKS_KEY_COMPACT=0"),
                                                         (20, 10, 10, 41, "CKKS_HYB_RS=0"),
                                                         (20, 10, 10, 41, "CKKS_HYB_FUSED_IP=0"),
                                                         (20, 10, 10, 41, "CKKS_CONV_V2=1")])
def test_hybrid_f64_specials_bit_exact(oracle_mod, monkeypatch, L, alpha, K, sp_bits, variant):
    """Special primes below 2^42 (FP64-mode: the ModUp special slots, the ModDown INTT and the
    fused ModDown + rescale conversion run on the FP64 pipe), P > Q_D with K = alpha 41-bit primes
    over 40-bit digits -- 40-bit special primes (drawn first, so above every q_i) also make every
    key limb compact (5-byte rows); mul_relin, the fused mul_relin_rescale and rotation vs the
    oracle; also with each hybrid kernel-variant switch (README) flipped."""
    from paper_1908_06972_b200 import ckks
    if variant:
        monkeypatch.setenv(*variant.split("="))
    bits = [40] * L
    p = oracle_mod.toy_params(12, bits, sp_bits, alpha=alpha, n_special=K)
    ctx = ckks.Context(12, bits, sp_bits, 2.0 ** 20, n_special=K, digit_limbs=alpha)
    assert ctx.q == p.q and ctx.special == p.special
    assert all(2 ** (sp_bits - 1) < x < 2 ** sp_bits for x in p.special)
    assert min(p.special) > max(p.q)  # P > Q_D for every digit (H3)
    kr = synth.KeyRandomness(11, p.log_n, p.q, p.P)
    rlk = oracle_mod.keygen_relin(p, kr.s, *kr.switch_key(0, dnum=p.dnum, special=p.special))
    kappa, gk = oracle_mod.keygen_galois(p, kr.s, 1, *kr.switch_key(7, dnum=p.dnum, special=p.special))
    ctx.import_switch_key(0, 0, _cuda(rlk))
    ctx.import_switch_key(1, 1, _cuda(gk))
    for level in (L, L - 1, 2):
        a, b = rand_ct(p, 2, level, 60 + level), rand_ct(p, 2, level, 70 + level)
        A, B = ctx.import_coeffs(_cuda(a), level, 1.0), ctx.import_coeffs(_cuda(b), level, 1.0)
        got = _host(ctx.export_coeffs(ctx.mul_relin(A, B)))
        got_f = _host(ctx.export_coeffs(ctx.mul_relin_rescale(A, B)))
        got_r = _host(ctx.export_coeffs(ctx.rotate(A, 1)))
        for c in range(2):
            oa = oracle_mod.Ciphertext([a[c, 0], a[c, 1]], level, 1.0)
            want = oracle_mod.mul_relin(p, oa, oracle_mod.Ciphertext([b[c, 0], b[c, 1]], level, 1.0), rlk)
            wr = oracle_mod.rescale(p, want)
            wrot = oracle_mod.apply_galois(p, oa, kappa, gk)
            for k in range(2):
                assert np.array_equal(got[c, k], want.c[k]), (level, c, k)
                assert np.array_equal(got_f[c, k], wr.c[k]), (level, c, k)
                assert np.array_equal(got_r[c, k], wrot.c[k]), (level, c, k)
    ctx.close()
