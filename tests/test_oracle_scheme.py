"""Pins for the oracle's scheme layer: encode/decode, enc/dec, HMult, rotation,
TotalSum and the PrivFT composer (run with -m "not gpu")."""
import json
import math
import os

import mpmath
import numpy as np
import pytest

from paper_1908_06972_b200 import synth
from tests import bigint_ref as ref

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))
T2 = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "table2_rotation.json")))


def _roots(log_n):
    n = 1 << log_n
    return [pow(5, j, 2 * n) for j in range(n // 2)]


def test_encode_matches_direct_evaluation(oracle_mod):
    """m(zeta^{5^j}) = Delta z_j up to the coefficient rounding (|err| <= N/2),
    evaluated directly in 50-digit arithmetic (reading A12)."""
    mpmath.mp.dps = 50
    log_n, scale = 6, 2.0 ** 30
    n = 1 << log_n
    z = synth.real_slots(synth.rng(1), n // 2) + 1j * synth.real_slots(synth.rng(2), n // 2)
    m = oracle_mod.encode_coeffs(z, scale, log_n)
    for j, r in enumerate(_roots(log_n)):
        zeta_r = mpmath.exp(1j * mpmath.pi * r / n)
        val = mpmath.fsum(int(m[k]) * zeta_r ** k for k in range(n))
        assert abs(val - scale * complex(z[j])) <= n / 2
    # decode of the same integers against the direct evaluation
    d = oracle_mod.decode_coeffs(m, scale, log_n)
    for j, r in enumerate(_roots(log_n)):
        zeta_r = mpmath.exp(1j * mpmath.pi * r / n)
        val = mpmath.fsum(int(m[k]) * zeta_r ** k for k in range(n)) / scale
        assert abs(complex(val) - d[j]) < 1e-9


def test_encode_constant_is_constant_poly(oracle_mod):
    """encoding a constant vector gives the constant polynomial round(Delta c)."""
    m = oracle_mod.encode_coeffs(np.full(512, 0.375), 2.0 ** 30, 10)
    assert m[0] == round(0.375 * 2 ** 30) and not np.any(m[1:])


def test_encode_roundtrip_bound(oracle_mod):
    log_n, scale = 13, 2.0 ** 40
    z = synth.real_slots(synth.rng(3), 1 << (log_n - 1))
    back = oracle_mod.decode_coeffs(oracle_mod.encode_coeffs(z, scale, log_n), scale, log_n)
    assert np.max(np.abs(back - z)) <= (1 << log_n) * 2.0 ** -41


def _small_scheme(oracle_mod, log_n=4, bits=(40, 30, 30), scale=2.0 ** 20, seed=3):
    p = oracle_mod.toy_params(log_n, list(bits), 60, scale)
    kr = synth.KeyRandomness(seed, p.log_n, p.q, p.P)
    pk = oracle_mod.keygen_public(p, kr.s, kr.pk_a, kr.pk_e)
    return p, kr, pk


def test_keygen_and_encrypt_exact_identity(oracle_mod):
    """P:139/P:141/P:142 with reading A1: c0 + c1 s = mu + e u + e0 + e1 s exactly over Z
    (schoolbook big-integer evaluation), with b = -a s + e."""
    p, kr, pk = _small_scheme(oracle_mod)
    z = synth.real_slots(synth.rng(5), p.slots)
    pt = oracle_mod.encode(p, z)
    u, e0, e1 = kr.enc(0)
    ct = oracle_mod.encrypt(p, pk, pt, u, e0, e1)
    dec = oracle_mod.decrypt(p, kr.s, ct)
    Q = math.prod(p.q)
    got = oracle_mod.centered(oracle_mod.crt_int(dec.m, p.q), Q)
    mu = oracle_mod.centered(oracle_mod.crt_int(pt.m, p.q), Q)
    want = [a + b + c + d for a, b, c, d in zip(mu, ref.negacyclic_mul_int(kr.pk_e, u), e0,
                                               ref.negacyclic_mul_int(e1, kr.s))]
    assert got == want


def test_three_part_decrypt_identity(oracle_mod):
    """P9: (c0 + c1 s)(c0' + c1' s) == d0 + d1 s + d2 s^2 mod Q exactly."""
    p, kr, pk = _small_scheme(oracle_mod)
    cts = []
    for tag in range(2):
        pt = oracle_mod.encode(p, synth.real_slots(synth.rng(10 + tag), p.slots))
        cts.append(oracle_mod.encrypt(p, pk, pt, *kr.enc(tag)))
    t = oracle_mod.tensor(p, cts[0], cts[1])
    dec3 = oracle_mod.decrypt(p, kr.s, t)
    a = oracle_mod.decrypt(p, kr.s, cts[0]).m
    b = oracle_mod.decrypt(p, kr.s, cts[1]).m
    assert np.array_equal(dec3.m, oracle_mod.poly_mul(a, b, p.mods(p.L), p.log_n))
    # and against schoolbook over the CRT integers
    Q = math.prod(p.q)
    ai, bi = oracle_mod.crt_int(a, p.q), oracle_mod.crt_int(b, p.q)
    assert oracle_mod.crt_int(dec3.m, p.q) == [x % Q for x in ref.negacyclic_mul_int(ai, bi)]


@pytest.fixture(scope="module")
def c1_world(oracle_mod):
    p = oracle_mod.preset("C1")
    kr = synth.KeyRandomness(1, p.log_n, p.q, p.P)
    pk = oracle_mod.keygen_public(p, kr.s, kr.pk_a, kr.pk_e)
    a, e = kr.switch_key(0)
    rlk = oracle_mod.keygen_relin(p, kr.s, a, e)
    gk = {}
    for st in (1, 4, 16, 64, 256, 1024, 2, 8):
        kappa, key = oracle_mod.keygen_galois(p, kr.s, st, *kr.switch_key(100 + st))
        gk[kappa] = key
    za = synth.real_slots(synth.rng(2), p.slots)
    zb = synth.real_slots(synth.rng(3), p.slots)
    ca = oracle_mod.encrypt(p, pk, oracle_mod.encode(p, za), *kr.enc(0))
    cb = oracle_mod.encrypt(p, pk, oracle_mod.encode(p, zb), *kr.enc(1))
    return dict(p=p, kr=kr, pk=pk, rlk=rlk, gk=gk, za=za, zb=zb, ca=ca, cb=cb)


def eps(p, floors=0, scale=None, fresh=2):
    """Semantic tolerance derived from the arithmetic.
    Fresh noise e*u + e0 + e1*s with BINARY u, s (readings A1, A2): e*u contains
    e*(1/2)(1 + X + ... ) whose coefficients are a random walk, concentrating
    ~ sigma N^1.5 / pi in the lowest slots; we allow 4 sigma N^1.5 / Delta per fresh
    input.  Per floor division (rescale Eq. 1 / A4, ModDown A7) the dropped fraction
    r0 + r1*s has |coefficient| <= 1 + HW(s) <= N + 1, so |slot error| <= N(N+1)/scale."""
    scale = p.scale if scale is None else scale
    return fresh * 4 * 3.2 * p.N ** 1.5 / p.scale + floors * p.N * (p.N + 1) / scale


def _dec(oracle_mod, w, ct):
    return oracle_mod.decode(w["p"], oracle_mod.decrypt(w["p"], w["kr"].s, ct)).real


def test_c1_hmult_relin_rescale_semantics(oracle_mod, c1_world):
    w = c1_world
    p = w["p"]
    out = oracle_mod.rescale(p, oracle_mod.mul_relin(p, w["ca"], w["cb"], w["rlk"]))
    assert out.level == p.L - 1
    assert out.scale == p.scale * p.scale / p.q[-1]
    err = np.max(np.abs(_dec(oracle_mod, w, out) - w["za"] * w["zb"]))
    assert err <= eps(p, floors=2, scale=out.scale), err


def test_c1_add_mulplain_semantics(oracle_mod, c1_world):
    w = c1_world
    p = w["p"]
    s = oracle_mod.add(p, w["ca"], w["cb"])
    assert np.max(np.abs(_dec(oracle_mod, w, s) - (w["za"] + w["zb"]))) <= eps(p)
    pt = oracle_mod.encode(p, w["zb"])
    m = oracle_mod.rescale(p, oracle_mod.mul_plain(p, w["ca"], pt))
    assert np.max(np.abs(_dec(oracle_mod, w, m) - w["za"] * w["zb"])) <= eps(p, floors=1, scale=m.scale)
    ap = oracle_mod.add_plain(p, w["ca"], pt)
    assert np.max(np.abs(_dec(oracle_mod, w, ap) - (w["za"] + w["zb"]))) <= eps(p)


def test_c1_rotation_is_cyclic_shift(oracle_mod, c1_world):
    """rotate by pi shifts decoded slots left by pi; 1365 is the HHW step (A10)."""
    w = c1_world
    p = w["p"]
    for st in (1, 1365):
        r = oracle_mod.rotate(p, w["ca"], st, w["gk"])
        nks = len(oracle_mod.rotation_steps(p, st))
        assert np.max(np.abs(_dec(oracle_mod, w, r) - np.roll(w["za"], -st))) <= eps(p, floors=nks)
    # rotate(rotate(a, 1), 1) == rotate(a, 2)
    r11 = oracle_mod.rotate(p, oracle_mod.rotate(p, w["ca"], 1, w["gk"]), 1, w["gk"])
    r2 = oracle_mod.rotate(p, w["ca"], 2, w["gk"])
    assert np.max(np.abs(_dec(oracle_mod, w, r11) - _dec(oracle_mod, w, r2))) <= 2 * eps(p, floors=2)


def test_rotation_count_matches_table2(oracle_mod):
    """P14: Table 2 HHW/LHW ratios equal the maximum number of signed
    power-of-two rotations over all steps in [0, N/2) (P:431 'log2 N / 2 at most')."""
    ratios = [h / l for h, l in zip(T2["rotate_hhw_ms"], T2["rotate_lhw_ms"])]
    for log_n, ratio, want in zip(T2["log_n"], ratios, T2["max_rotations_expected"]):
        p = oracle_mod.Params(log_n, [97], 0, 1.0)
        worst = max(len(oracle_mod.rotation_steps(p, s)) for s in range(p.slots))
        assert worst == want
        assert abs(ratio - worst) < 0.25, (log_n, ratio, worst)
        binary_worst = log_n - 1
        assert abs(ratio - binary_worst) > 3


def test_total_sum_worked_example(oracle_mod):
    """(1,2,3,4) at t = 4 -> (10,10,10,10); e_0 -> all ones."""
    p = oracle_mod.toy_params(3, [40, 30], 60, 2.0 ** 20)
    kr = synth.KeyRandomness(4, p.log_n, p.q, p.P)
    pk = oracle_mod.keygen_public(p, kr.s, kr.pk_a, kr.pk_e)
    gk = dict(oracle_mod.keygen_galois(p, kr.s, st, *kr.switch_key(st)) for st in (1, 2))
    for v, want in ((GOLD["total_sum"]["v"], [10.0] * 4), ([1, 0, 0, 0], [1.0] * 4)):
        ct = oracle_mod.encrypt(p, pk, oracle_mod.encode(p, v), *kr.enc(0))
        out = oracle_mod.total_sum(p, ct, gk)
        got = oracle_mod.decode(p, oracle_mod.decrypt(p, kr.s, out)).real
        assert np.max(np.abs(got - want)) < 1e-3


def test_softmax_polynomial_values(oracle_mod):
    """P:260 / S:324-326: X^2/8 + X/2 + 1/4 at 0, 2, -2, evaluated encrypted exactly as
    the composer does ((s^2 + 4 s + 2) / 8 with one mul_relin and one rescale)."""
    p = oracle_mod.toy_params(5, [60, 40, 40], 60, 2.0 ** 30)
    kr = synth.KeyRandomness(8, p.log_n, p.q, p.P)
    pk = oracle_mod.keygen_public(p, kr.s, kr.pk_a, kr.pk_e)
    rlk = oracle_mod.keygen_relin(p, kr.s, *kr.switch_key(0))
    xs = [c[0] for c in GOLD["softmax_poly"]["cases"]]
    want = [c[1] for c in GOLD["softmax_poly"]["cases"]]
    s = oracle_mod.encrypt(p, pk, oracle_mod.encode(p, xs, level=2), *kr.enc(0))
    sq = oracle_mod.mul_relin(p, s, s, rlk)
    g = oracle_mod.rescale(p, oracle_mod.add(p, sq, oracle_mod.mul_const(p, s, 4.0, s.scale)))
    g = oracle_mod.add_const(p, g, 2.0)
    g = oracle_mod.Ciphertext(g.c, g.level, g.scale * 8)
    got = oracle_mod.decode(p, oracle_mod.decrypt(p, kr.s, g)).real[:3]
    assert np.max(np.abs(got - want)) < 1e-4
    assert np.allclose(oracle_mod.fasttext_plain(np.eye(3), 1, np.eye(3), np.diag(xs), True).diagonal(), want)


def test_message_count():
    g = GOLD["message_count"]
    assert math.ceil(g["m"] / g["t"]) == g["chunks"] == 123


def _privft_case(oracle_mod, log_n, m, n, c, seed, poly, H=None, O=None, v=None, w=None):
    qs, sp = oracle_mod.prime_chain(log_n, [60, 40, 40, 40, 40])
    p = oracle_mod.Params(log_n, qs, sp[0], 2.0 ** 40)
    t = p.slots
    K = -(-m // t)
    g = synth.rng(seed)
    H = g.uniform(-1, 1, (m, n)) if H is None else H
    O = g.uniform(-1, 1, (n, c)) if O is None else O
    if v is None:
        v, w = synth.bag(g, m, 60)
    kr = synth.KeyRandomness(seed, p.log_n, p.q, p.P)
    pk = oracle_mod.keygen_public(p, kr.s, kr.pk_a, kr.pk_e)
    rlk = oracle_mod.keygen_relin(p, kr.s, *kr.switch_key(0))
    gk = dict(oracle_mod.keygen_galois(p, kr.s, 1 << i, *kr.switch_key(1 + i)) for i in range(log_n - 1))
    vp = np.zeros(K * t)
    vp[:m] = v
    chunks = [oracle_mod.encrypt(p, pk, oracle_mod.encode(p, vp[k * t:(k + 1) * t]), *kr.enc(k)) for k in range(K)]
    Hp = np.zeros((K * t, n))
    Hp[:m] = H
    H_pts = [[oracle_mod.encode(p, Hp[k * t:(k + 1) * t, j]) for k in range(K)] for j in range(n)]
    O_pts = [oracle_mod.encode(p, O[j], level=p.L - 2) for j in range(n)]
    out = oracle_mod.privft_infer(p, chunks, w, H_pts, O_pts, rlk, gk, poly)
    got = oracle_mod.decode(p, oracle_mod.decrypt(p, kr.s, out)).real[:c]
    want = oracle_mod.fasttext_plain(v, w, H, O, poly)
    return p, out, got, want


@pytest.mark.parametrize("poly", [False, True])
def test_privft_matches_float64_fasttext(oracle_mod, poly):
    """P12: decrypted scores == float64 Alg "fasttext Inference" steps 2-3 (+ the
    polynomial), argmax equal; depth = 3 (4) rescales from L = 5 (P16)."""
    p, out, got, want = _privft_case(oracle_mod, 10, 1300, 4, 3, 21, poly)
    assert out.level == p.L - (4 if poly else 3)
    assert np.max(np.abs(got - want)) < 1e-4, (got, want)
    assert np.argmax(got) == np.argmax(want)


def test_privft_identity_model(oracle_mod):
    """S:316-style identity case: m = n = c, H = O = I -> s = v / w."""
    v = np.array([3.0, 1.0, 0.0, 2.0])
    p, out, got, want = _privft_case(oracle_mod, 10, 4, 4, 4, 5, False, H=np.eye(4), O=np.eye(4), v=v, w=6)
    assert np.max(np.abs(got - v / 6)) < 1e-6


def test_privft_infer_workers_identical(oracle_mod):
    """The column-parallel map (workers > 1, timing only) is the same arithmetic."""
    p = oracle_mod.toy_params(10, [60, 40, 40, 40, 40], 60, scale=2.0 ** 40)
    g = synth.rng(77)
    kr = synth.KeyRandomness(77, p.log_n, p.q, p.P)
    rlk = oracle_mod.keygen_relin(p, kr.s, *kr.switch_key(0))
    gk = dict(oracle_mod.keygen_galois(p, kr.s, 1 << i, *kr.switch_key(1 + i)) for i in range(p.log_n - 1))
    K, n = 2, 3
    H = [[oracle_mod.Plaintext(synth.uniform_residues(g, p.q, p.N), p.L, p.scale) for _ in range(K)]
         for _ in range(n)]
    O = [oracle_mod.Plaintext(synth.uniform_residues(g, p.q[:p.L - 2], p.N), p.L - 2, p.scale) for _ in range(n)]
    bag = [oracle_mod.Ciphertext([synth.uniform_residues(g, p.q, p.N) for _ in range(2)], p.L, p.scale)
           for _ in range(K)]
    a = oracle_mod.privft_infer(p, bag, 37, H, O, rlk, gk, True)
    b = oracle_mod.privft_infer(p, bag, 37, H, O, rlk, gk, True, workers=3)
    assert a.level == b.level and a.scale == b.scale
    assert all(np.array_equal(x, y) for x, y in zip(a.c, b.c))
