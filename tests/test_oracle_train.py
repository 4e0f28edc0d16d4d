"""Pins for the oracle's encrypted training step: the decrypted updated
model matches the float64 minibatch gradient step, and the level ledger is 9 per minibatch
(P:487).  -m "not gpu"."""
import numpy as np
import pytest

from paper_1908_06972_b200 import synth


def _setup(oracle_mod, log_n=10, m=300, n=3, c=2, E=2, seed=3):
    p = oracle_mod.toy_params(log_n, [60] + [40] * 10, 60, scale=2.0 ** 40)
    t = p.slots
    kr = synth.KeyRandomness(seed, p.log_n, p.q, p.P)
    pk = oracle_mod.keygen_public(p, kr.s, kr.pk_a, kr.pk_e)
    rlk = oracle_mod.keygen_relin(p, kr.s, *kr.switch_key(0))
    gk = dict(oracle_mod.keygen_galois(p, kr.s, 1 << i, *kr.switch_key(1 + i)) for i in range(log_n - 1))
    g = synth.rng(seed)
    H = g.uniform(-1, 1, (m, n))
    O = g.uniform(-1, 1, (n, c))
    enc = lambda z, tag: oracle_mod.encrypt(p, pk, oracle_mod.encode(p, z), *kr.enc(tag))
    Hc = [enc(np.pad(H[:, j], (0, t - m)), 100 + j) for j in range(n)]
    Oc = [enc(np.pad(O[j], (0, t - c)), 200 + j) for j in range(n)]
    exs, plain = [], []
    for k in range(E):
        v, w = synth.bag(synth.rng(50 + k), m, 40)
        y = k % c
        exs.append((enc(np.pad(v, (0, t - m)), 300 + k), w, y))
        plain.append((v, w, y))
    return p, kr, rlk, gk, H, O, Hc, Oc, exs, plain


def test_train_step_matches_float64(oracle_mod):
    p, kr, rlk, gk, H, O, Hc, Oc, exs, plain = _setup(oracle_mod)
    eta, c = 0.5, O.shape[1]
    GH, GO = oracle_mod.train_gradients(p, Hc, Oc, exs, c, rlk, gk)
    Hn, On = oracle_mod.train_update(p, Hc, Oc, GH, GO, eta)
    assert Hn[0].level == p.L - 9 and On[0].level == p.L - 9  # 9 levels per minibatch
    Hw, Ow = oracle_mod.train_plain(H, O, plain, c, eta)
    m = H.shape[0]
    dec = lambda ct: oracle_mod.decode(p, oracle_mod.decrypt(p, kr.s, ct)).real
    for j in range(H.shape[1]):
        assert np.max(np.abs(dec(Hn[j])[:m] - Hw[:, j])) < 1e-4
        assert np.max(np.abs(dec(On[j])[:c] - Ow[j])) < 1e-4
    # the step actually moved the model (gradient not vanishing at this size)
    assert np.max(np.abs(Hw - H)) > 1e-3


def test_eta_zero_is_identity(oracle_mod):
    p, kr, rlk, gk, H, O, Hc, Oc, exs, plain = _setup(oracle_mod, E=1)
    GH, GO = oracle_mod.train_gradients(p, Hc, Oc, exs, O.shape[1], rlk, gk)
    Hn, On = oracle_mod.train_update(p, Hc, Oc, GH, GO, 0.0)
    dec = lambda ct: oracle_mod.decode(p, oracle_mod.decrypt(p, kr.s, ct)).real
    assert np.max(np.abs(dec(Hn[0])[:H.shape[0]] - H[:, 0])) < 1e-5
