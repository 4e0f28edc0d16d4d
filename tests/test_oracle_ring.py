"""Pins for the oracle's exact ring arithmetic (run with -m "not gpu").

Each test ties an oracle function to something other than itself: brute force,
Python big integers, schoolbook convolution, the direct NTT sum, or a worked
example from the paper/SPEC (tests/golden/worked_examples.json)."""
import json
import math
import os
import random

import numpy as np
import pytest

from tests import bigint_ref as ref

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


def test_is_prime_matches_trial_division(oracle_mod):
    for n in range(0, 20000):
        assert oracle_mod.is_prime(n) == ref._trial(n), n


def test_is_prime_large_composites_and_primes(oracle_mod):
    rnd = random.Random(5)
    for _ in range(40):
        p = rnd.randrange(1 << 40, 1 << 61) | 1
        assert oracle_mod.is_prime(p) == ref.prove_prime(p)
    # strong pseudoprimes to several small bases must be rejected
    for n in [3215031751, 2152302898747, 3474749660383, 341550071728321, 3825123056546413051]:
        assert not oracle_mod.is_prime(n)


def test_prime_scan_toy_example(oracle_mod):
    """S:54 claims 17; brute force says 29 (largest prime < 32 that is 1 mod 4)."""
    g = GOLD["prime_chain_toy"]
    brute = max(x for x in range(2, 1 << g["bits"]) if x % (2 * g["N"]) == 1 and ref._trial(x))
    assert brute == g["value"] == 29
    assert oracle_mod.prime_scan(1, g["bits"], 0, 1) == [29]


@pytest.mark.parametrize("log_n,bits,count", [(12, 30, 4), (13, 40, 5), (16, 40, 31), (13, 60, 2), (16, 60, 1)])
def test_prime_scan_no_skips(oracle_mod, log_n, bits, count):
    """Scan = every prime = 1 mod 2N below 2^bits in decreasing order: each hit has a
    Lucas primality certificate, and every skipped candidate has a Fermat witness."""
    got = oracle_mod.prime_scan(log_n, bits, 0, count)
    two_n = 2 << log_n
    x = ((1 << bits) - 2) // two_n * two_n + 1
    for p in got:
        assert p % two_n == 1 and p < (1 << bits)
        assert ref.prove_prime(p)
        while x > p:  # candidates strictly between
            assert any(pow(a, x - 1, x) != 1 for a in (2, 3, 5, 7)) or x % 3 == 0 or not ref.prove_prime(x)
            x -= two_n
        x -= two_n
    assert got == sorted(got, reverse=True)


def test_appendix_c_chains(oracle_mod):
    """The presets re-derive SURVEY Appendix C (written there by the same O1 rule)."""
    c1 = oracle_mod.preset("C1")
    assert c1.P == 1152921504606830593 and c1.q == [1073692673, 1073668097, 1073651713]
    c4 = oracle_mod.preset("C4")
    assert c4.P == 1152921504606830593
    assert c4.q == [1152921504606748673, 1099511480321, 1099510890497, 1099510824961, 1099510054913]
    c3 = oracle_mod.preset("C3")
    assert c3.P == 1152921504606584833 and len(c3.q) == 30
    assert c3.q[0] == 1099510054913 and c3.q[-1] == 1099457495041


@pytest.mark.parametrize("q,log_n", [(17, 3), (97, 4), (257, 7), (7681, 8)])
def test_min_psi_brute_force(oracle_mod, q, log_n):
    n = 1 << log_n
    roots = [g for g in range(2, q) if pow(g, n, q) == q - 1]
    assert oracle_mod.min_psi(q, log_n) == min(roots)


@pytest.mark.parametrize("log_n", [2, 3, 6, 8])
def test_ntt_equals_direct_definition(oracle_mod, log_n):
    q = oracle_mod.prime_scan(log_n, 30, 0, 1)[0]
    psi = oracle_mod.min_psi(q, log_n)
    rnd = np.random.default_rng(log_n)
    a = rnd.integers(0, q, 1 << log_n, dtype=np.uint64)
    assert oracle_mod.ntt_fwd(a, log_n, q, psi).tolist() == ref.direct_ntt(a.tolist(), q, psi)


@pytest.mark.parametrize("log_n,bits", [(12, 30), (13, 60), (16, 40)])
def test_ntt_roundtrip_exact(oracle_mod, log_n, bits):
    q = oracle_mod.prime_scan(log_n, bits, 0, 1)[0]
    a = np.random.default_rng(1).integers(0, q, 1 << log_n, dtype=np.uint64)
    assert np.array_equal(oracle_mod.ntt_inv(oracle_mod.ntt_fwd(a, log_n, q), log_n, q), a)


def test_spec_ntt_examples(oracle_mod):
    q = oracle_mod.prime_scan(2, 30, 0, 1)[0]
    g = GOLD["ntt_square"]
    assert oracle_mod.poly_mul([g["a"]], [g["a"]], [q], 2)[0].tolist() == g["product"]
    g = GOLD["ntt_wrap"]
    out = oracle_mod.poly_mul([g["a"]], [g["b"]], [q], 2)[0].tolist()
    assert out == [x % q for x in g["product_signed"]]


@pytest.mark.parametrize("log_n", [3, 5, 6])
def test_poly_mul_schoolbook(oracle_mod, log_n):
    mods = oracle_mod.prime_scan(log_n, 60, 0, 2) + oracle_mod.prime_scan(log_n, 30, 0, 1)
    rnd = np.random.default_rng(7)
    a = np.stack([rnd.integers(0, q, 1 << log_n, dtype=np.uint64) for q in mods])
    b = np.stack([rnd.integers(0, q, 1 << log_n, dtype=np.uint64) for q in mods])
    out = oracle_mod.poly_mul(a, b, mods, log_n)
    for i, q in enumerate(mods):
        assert out[i].tolist() == ref.negacyclic_mul(a[i].tolist(), b[i].tolist(), q)


def test_add_sub_neg_scalar(oracle_mod):
    mods = oracle_mod.prime_scan(4, 40, 0, 3)
    rnd = np.random.default_rng(3)
    a = np.stack([rnd.integers(0, q, 16, dtype=np.uint64) for q in mods])
    b = np.stack([rnd.integers(0, q, 16, dtype=np.uint64) for q in mods])
    c = np.array([rnd.integers(0, q) for q in mods], dtype=np.uint64)
    s = oracle_mod.poly_add(a, b, mods, 4)
    d = oracle_mod.poly_sub(a, b, mods, 4)
    ng = oracle_mod.poly_neg(a, mods, 4)
    sc = oracle_mod.poly_scalar_mul(a, c, mods, 4)
    for i, q in enumerate(mods):
        for k in range(16):
            x, y = int(a[i, k]), int(b[i, k])
            assert int(s[i, k]) == (x + y) % q
            assert int(d[i, k]) == (x - y) % q
            assert int(ng[i, k]) == (-x) % q
            assert int(sc[i, k]) == (x * int(c[i])) % q
    e = np.array([-19, -1, 0, 1, 19] + [0] * 11, dtype=np.int64)
    r = oracle_mod.poly_from_signed(e, mods, 4)
    for i, q in enumerate(mods):
        assert [int(v) for v in r[i]] == [int(v) % q for v in e]


def test_crt_example(oracle_mod):
    g = GOLD["crt"]
    assert oracle_mod.crt_int(np.array([[g["residues"][0]], [g["residues"][1]]]), g["mods"]) == [g["value"]]
    assert ref.crt(g["residues"], g["mods"]) == g["value"]


def test_rescale_exhaustive_toy_chain(oracle_mod):
    """Eq. (1) limb formula == big-integer floor(c / q_last), every c in [0, 13*11)."""
    mods = GOLD["rescale"]["mods"]
    Q = math.prod(mods)
    for c in range(Q):
        limbs = np.array([[c % mods[0]], [c % mods[1]]], dtype=np.uint64)
        out = oracle_mod.rescale_poly(limbs, mods, 0)
        assert int(out[0, 0]) == (c // mods[1]) % mods[0]
    for c, want in GOLD["rescale"]["cases"]:
        limbs = np.array([[c % mods[0]], [c % mods[1]]], dtype=np.uint64)
        assert int(oracle_mod.rescale_poly(limbs, mods, 0)[0, 0]) == want


def test_rescale_matches_bigint_floor_real_primes(oracle_mod):
    p = oracle_mod.preset("C4")
    mods = p.q
    rnd = np.random.default_rng(11)
    c = np.stack([rnd.integers(0, q, 64, dtype=np.uint64) for q in mods])
    out = oracle_mod.rescale_poly(c, mods, 6)
    ints = oracle_mod.crt_int(c, mods)
    for k in range(64):
        fl = ints[k] // mods[-1]
        assert [int(out[i, k]) for i in range(4)] == [fl % q for q in mods[:4]]


def test_automorphism_examples(oracle_mod):
    g = GOLD["automorphism"]
    q = oracle_mod.prime_scan(2, 30, 0, 1)[0]
    assert oracle_mod.automorphism([g["a"]], g["kappa"], [q], 2)[0].tolist() == g["out"]
    log_n = 4
    mods = oracle_mod.prime_scan(log_n, 40, 0, 2)
    rnd = np.random.default_rng(2)
    a = np.stack([rnd.integers(0, q, 16, dtype=np.uint64) for q in mods])
    b = np.stack([rnd.integers(0, q, 16, dtype=np.uint64) for q in mods])
    for kappa in (1, 3, 5, 25, 31, 2 * 16 - 1):
        out = oracle_mod.automorphism(a, kappa, mods, log_n)
        for i, q in enumerate(mods):
            assert out[i].tolist() == [x % q for x in ref.substitute(a[i].tolist(), kappa)]
        # ring homomorphism
        lhs = oracle_mod.automorphism(oracle_mod.poly_mul(a, b, mods, log_n), kappa, mods, log_n)
        rhs = oracle_mod.poly_mul(oracle_mod.automorphism(a, kappa, mods, log_n),
                                  oracle_mod.automorphism(b, kappa, mods, log_n), mods, log_n)
        assert np.array_equal(lhs, rhs)


def _toy(oracle_mod, log_n=3, bits=(30, 30, 30)):
    return oracle_mod.toy_params(log_n, list(bits), 40)


def test_keyswitch_bruteforce_bigint(oracle_mod):
    """P5: the whole key switch (ModUp lift A8, inner product, floor ModDown A7) equals
    a Python big-integer evaluation over the integer basis Q*P at N = 8."""
    p = _toy(oracle_mod)
    n, L = p.N, p.L
    rnd = np.random.default_rng(4)
    em = p.q + [p.P]
    key = np.stack([np.stack([np.stack([rnd.integers(0, q, n, dtype=np.uint64) for q in em]) for _ in range(2)])
                    for _ in range(L)])
    for level in (L, 2):
        d = np.stack([rnd.integers(0, q, n, dtype=np.uint64) for q in p.q[:level]])
        k0, k1 = oracle_mod.keyswitch(d, key, L, em, p.log_n)
        basis = p.q[:level] + [p.P]
        QP = math.prod(basis)
        for part, got in ((0, k0), (1, k1)):
            acc = [0] * n
            for j in range(level):
                dj = [int(x) for x in d[j]]  # unsigned representative in [0, q_j)
                kj = [ref.crt([int(key[j, part, (i if i < level else L), k]) for i in range(level + 1)], basis)
                      for k in range(n)]
                prod = ref.negacyclic_mul_int(dj, kj)
                acc = [(x + y) % QP for x, y in zip(acc, prod)]
            fl = [x // p.P for x in acc]
            for i in range(level):
                assert got[i].tolist() == [v % p.q[i] for v in fl]


def test_keyswitch_identity_with_real_key(oracle_mod):
    """P6: with a key for s_from -> s, k0 + k1 s = d s_from + noise, |noise| <= N + 2
    (Sum_j d~_j e_j / P < 1 at these sizes; the two floors add at most 1 + ||s||_1)."""
    from paper_1908_06972_b200 import synth
    p = oracle_mod.toy_params(10, [30, 30, 30], 60)
    kr = synth.KeyRandomness(9, p.log_n, p.q, p.P)
    a, e = kr.switch_key(0)
    em = p.ext_mods()
    s_from = synth.uniform_residues(synth.rng(3), list(em), p.N)  # arbitrary source key
    key = oracle_mod.keygen_switch(p, kr.s, s_from, a, e)
    d = synth.uniform_residues(synth.rng(4), p.q, p.N)
    k0, k1 = oracle_mod.keyswitch(d, key, p.L, em, p.log_n)
    mods = p.mods(p.L)
    s_r = oracle_mod.poly_from_signed(kr.s, mods, p.log_n)
    lhs = oracle_mod.poly_add(k0, oracle_mod.poly_mul(k1, s_r, mods, p.log_n), mods, p.log_n)
    rhs = oracle_mod.poly_mul(d, s_from[: p.L], mods, p.log_n)
    diff = oracle_mod.poly_sub(lhs, rhs, mods, p.log_n)
    Q = math.prod(p.q)
    err = oracle_mod.centered(oracle_mod.crt_int(diff, p.q), Q)
    assert max(abs(x) for x in err) <= p.N + 2
