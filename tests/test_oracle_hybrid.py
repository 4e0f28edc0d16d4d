"""Pins for the oracle's hybrid key switching (alpha-limb digits, K special
primes, HPS fast base conversion).  -m "not gpu"."""
import math

import numpy as np
import pytest

from paper_1908_06972_b200 import synth
from tests import bigint_ref as ref


@pytest.mark.parametrize("ns", [1, 2, 3, 5])
def test_fast_bconv_is_x_plus_small_multiple(oracle_mod, ns):
    """conv_D(x) = x + u Q_D with one integer 0 <= u < |D| shared by every target modulus
    (the defining property of fast base conversion); |D| = 1 is the exact lift (A8)."""
    src_m = oracle_mod.prime_scan(5, 30, 0, ns)
    tgt_m = oracle_mod.prime_scan(5, 40, 0, 3) + oracle_mod.prime_scan(5, 60, 0, 2)
    mods = src_m + tgt_m
    g = synth.rng(ns)
    x = synth.uniform_residues(g, src_m, 32)
    out = oracle_mod.fast_bconv(x, list(range(ns)), list(range(ns, len(mods))), mods, 5)
    QD = math.prod(src_m)
    for k in range(32):
        X = ref.crt([int(x[i, k]) for i in range(ns)], src_m)
        us = {((int(out[t, k]) - X) * pow(QD, -1, m)) % m for t, m in enumerate(tgt_m)}
        assert len(us) == 1
        u = us.pop()
        assert 0 <= u < ns
        if ns == 1:
            assert u == 0


def test_hybrid_with_alpha1_K1_equals_per_limb_keyswitch(oracle_mod):
    """alpha = K = 1 hybrid code path == or_keyswitch (itself pinned by big-int brute force)."""
    p = oracle_mod.toy_params(6, [30, 30, 30, 30], 60)
    g = synth.rng(2)
    em = p.ext_mods()
    key = np.stack([np.stack([synth.uniform_residues(g, list(em), p.N) for _ in range(2)]) for _ in range(p.L)])
    d = synth.uniform_residues(g, p.q, p.N)
    a = oracle_mod.keyswitch(d, key, p.L, em, p.log_n)
    lib = oracle_mod.lib()
    o0 = np.empty_like(d)
    o1 = np.empty_like(d)
    lib.or_keyswitch_hybrid(oracle_mod._p(d), p.L, oracle_mod._p(key), p.L, 1, 1, oracle_mod._p(em), p.log_n,
                            oracle_mod._p(o0), oracle_mod._p(o1))
    assert np.array_equal(a[0], o0) and np.array_equal(a[1], o1)


@pytest.mark.parametrize("alpha,K,level", [(3, 2, 6), (2, 2, 5), (4, 3, 6), (6, 2, 6), (3, 2, 4)])
def test_hybrid_keyswitch_identity(oracle_mod, alpha, K, level):
    """k0 + k1 s = d s_from + noise with |noise| <= sum_d |conv(d_d)| N 19 / P + (K+1)(N+1):
    the hybrid key (P Q^_d s_from per digit) and the fast-base-conversion ModUp/ModDown."""
    p = oracle_mod.toy_params(10, [30] * 6, 60, alpha=alpha, n_special=K)
    kr = synth.KeyRandomness(5, p.log_n, p.q, p.P)
    a, e = kr.switch_key(0, dnum=p.dnum, special=p.special)
    em = p.ext_mods()
    s_from = synth.uniform_residues(synth.rng(8), list(em), p.N)
    key = oracle_mod.keygen_switch(p, kr.s, s_from, a, e)
    assert key.shape == (p.dnum, 2, p.L + K, p.N)
    d = synth.uniform_residues(synth.rng(9), p.q[:level], p.N)
    k0, k1 = oracle_mod.keyswitch(d, key, p.L, em, p.log_n, alpha, K)
    mods = p.q[:level]
    s_r = oracle_mod.poly_from_signed(kr.s, mods, p.log_n)
    lhs = oracle_mod.poly_add(k0, oracle_mod.poly_mul(k1, s_r, mods, p.log_n), mods, p.log_n)
    rhs = oracle_mod.poly_mul(d, s_from[:level], mods, p.log_n)
    diff = oracle_mod.poly_sub(lhs, rhs, mods, p.log_n)
    err = max(abs(x) for x in oracle_mod.centered(oracle_mod.crt_int(diff, mods), math.prod(mods)))
    beta = -(-level // alpha)
    QD = max(math.prod(p.q[j * alpha:min(j * alpha + alpha, level)]) for j in range(beta))
    bound = beta * alpha * QD * p.N * 19 / p.P + (K + 1) * (p.N + 1)
    assert err <= bound, (err, bound)


def test_hybrid_hmult_semantics(oracle_mod):
    """decode(decrypt(rescale(mul_relin))) ~ a*b with a hybrid relinearisation key."""
    p = oracle_mod.toy_params(12, [40, 30, 30, 30], 60, scale=2.0 ** 30, alpha=2, n_special=2)
    kr = synth.KeyRandomness(11, p.log_n, p.q, p.P)
    pk = oracle_mod.keygen_public(p, kr.s, kr.pk_a, kr.pk_e)
    rlk = oracle_mod.keygen_relin(p, kr.s, *kr.switch_key(0, dnum=p.dnum, special=p.special))
    za = synth.real_slots(synth.rng(1), p.slots)
    zb = synth.real_slots(synth.rng(2), p.slots)
    ca = oracle_mod.encrypt(p, pk, oracle_mod.encode(p, za), *kr.enc(0))
    cb = oracle_mod.encrypt(p, pk, oracle_mod.encode(p, zb), *kr.enc(1))
    out = oracle_mod.rescale(p, oracle_mod.mul_relin(p, ca, cb, rlk))
    got = oracle_mod.decode(p, oracle_mod.decrypt(p, kr.s, out)).real
    tol = 2 * 4 * 3.2 * p.N ** 1.5 / p.scale + 3 * p.N * (p.N + 1) / out.scale
    assert np.max(np.abs(got - za * zb)) <= tol
