"""Full-size parity (BASELINE configs, the bench's launch configurations) and edge cases:
C3 HMult+relin+rescale (N = 2^16, l = 30) against the oracle on every output limb; PrivFT
at the full vocabulary (m = 500,000 -> K = 123 chunks) with the key switch forced through
many chunks; maximum L; degenerate rotations."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1908_06972_b200 import synth  # noqa: E402


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).cuda()


def _host(t):
    return t.cpu().numpy().view(np.uint64)


def test_c3_hmult_relin_rescale_full_vs_oracle(oracle_mod):
    """BASELINE metric op at its full size: every limb of both output polynomials."""
    from paper_1908_06972_b200 import ckks
    p = oracle_mod.preset("C3")
    ctx = ckks.Context(16, [40] * 30, 60, 2.0 ** 40)
    assert ctx.q == p.q and ctx.P == p.P
    g = synth.rng(16)
    em = list(p.ext_mods())
    rlk = np.stack([np.stack([synth.uniform_residues(g, em, p.N) for _ in range(2)]) for _ in range(p.L)])
    ctx.import_switch_key(0, 0, _cuda(rlk))
    a = np.stack([synth.uniform_residues(g, p.q, p.N) for _ in range(2)])[None]
    b = np.stack([synth.uniform_residues(g, p.q, p.N) for _ in range(2)])[None]
    A, B = ctx.import_coeffs(_cuda(a), 30, p.scale), ctx.import_coeffs(_cuda(b), 30, p.scale)
    got = _host(ctx.export_coeffs(ctx.rescale(ctx.mul_relin(A, B))))[0]
    want = oracle_mod.rescale(p, oracle_mod.mul_relin(p, oracle_mod.Ciphertext([a[0, 0], a[0, 1]], 30, p.scale),
                                                       oracle_mod.Ciphertext([b[0, 0], b[0, 1]], 30, p.scale), rlk))
    assert np.array_equal(got[0], want.c[0]) and np.array_equal(got[1], want.c[1])


@pytest.mark.parametrize("budget_mb", ["1", "1024"])
def test_c4_privft_full_vocabulary(oracle_mod, budget_mb, monkeypatch):
    """m = 500,000 (K = 123 chunks) at C4, 2 queries x 6 columns, bit-exact; the
    1 MiB budget forces the key switches through many small chunks."""
    from paper_1908_06972_b200 import ckks
    monkeypatch.setenv("CKKS_KS_BUDGET_MB", budget_mb)
    p = oracle_mod.preset("C4")
    ctx = ckks.Context(13, [60, 40, 40, 40, 40], 60, 2.0 ** 40)
    m, n, c, B = 500000, 6, 4, 2
    t = p.slots
    K = -(-m // t)
    assert K == 123
    g = synth.rng(44)
    kr = synth.KeyRandomness(44, p.log_n, p.q, p.P)
    rlk = oracle_mod.keygen_relin(p, kr.s, *kr.switch_key(0))
    ctx.import_switch_key(0, 0, _cuda(rlk))
    gk = {}
    for i in range(p.log_n - 1):
        kappa, key = oracle_mod.keygen_galois(p, kr.s, 1 << i, *kr.switch_key(1 + i))
        gk[kappa] = key
        ctx.import_switch_key(1, 1 << i, _cuda(key))
    # random residues stand in for the encoded model and the encrypted bags (exact ring ops)
    H_pts = [[oracle_mod.Plaintext(synth.uniform_residues(g, p.q, p.N), p.L, p.scale) for _ in range(K)]
             for _ in range(n)]
    O_pts = [oracle_mod.Plaintext(synth.uniform_residues(g, p.q[:p.L - 2], p.N), p.L - 2, p.scale) for _ in range(n)]
    bags = [[oracle_mod.Ciphertext([synth.uniform_residues(g, p.q, p.N) for _ in range(2)], p.L, p.scale)
             for _ in range(K)] for _ in range(B)]
    ws = [57, 411]
    Hd = ctx.import_coeffs(_cuda(np.stack([H_pts[j][k].m for j in range(n) for k in range(K)])[:, None]), p.L,
                           p.scale)
    Od = ctx.import_coeffs(_cuda(np.stack([o.m for o in O_pts])[:, None]), p.L - 2, p.scale)
    model = ctx.privft_model_wrap(Hd, Od, m, n, c)
    bag = ctx.import_coeffs(_cuda(np.stack([np.stack(ct.c) for q in bags for ct in q])), p.L, p.scale)
    out = ctx.privft_infer(model, bag, ws, True)
    got = _host(ctx.export_coeffs(out))
    for b in range(B):
        want = oracle_mod.privft_infer(p, bags[b], ws[b], H_pts, O_pts, rlk, gk, True)
        assert np.array_equal(got[b, 0], want.c[0]) and np.array_equal(got[b, 1], want.c[1]), b


def test_max_limbs_and_degenerate_rotations(oracle_mod):
    from paper_1908_06972_b200 import ckks
    ctx = ckks.Context(12, [50] * 60, 60, 2.0 ** 40)  # L = 60: the largest chain the ABI accepts
    assert len(ctx.q) == 60 and all(q < (1 << 50) for q in ctx.q)
    x = synth.uniform_residues(synth.rng(3), ctx.q, ctx.N)[None]
    tx = _cuda(x)
    ctx.ntt(tx)
    ctx.ntt(tx, inverse=True)
    assert np.array_equal(_host(tx), x)
    p = oracle_mod.preset("C1")
    c1 = ckks.Context(12, [30] * 3, 60, 2.0 ** 30)
    a = np.stack([synth.uniform_residues(synth.rng(5), p.q, p.N) for _ in range(2)])[None]
    A = c1.import_coeffs(_cuda(a), 3, 1.0)
    for steps in (0, p.slots, -p.slots, 3 * p.slots):  # identity rotations need no key (A31)
        assert np.array_equal(_host(c1.export_coeffs(c1.rotate(A, steps))), a)
    with pytest.raises(ckks.CkksError):
        c1.rotate(A, 1)  # no Galois key imported


def test_n15_hmult_and_rotate_vs_oracle(oracle_mod):
    """N = 2^15 (column phase B1 = 7, row phase B2 = 8: the only ring with unequal phases above
    2^13) at 6 x 40-bit limbs, two ciphertexts: HMult+relin+rescale and rotate(1) bit-exact."""
    from paper_1908_06972_b200 import ckks
    log_n, bits = 15, [40] * 6
    qs, sp = oracle_mod.prime_chain(log_n, bits)
    p = oracle_mod.Params(log_n, qs, sp[0], 2.0 ** 40)
    ctx = ckks.Context(log_n, bits, 60, 2.0 ** 40)
    assert ctx.q == p.q
    kr = synth.KeyRandomness(15, p.log_n, p.q, p.P)
    rlk = oracle_mod.keygen_relin(p, kr.s, *kr.switch_key(0))
    kappa, gk = oracle_mod.keygen_galois(p, kr.s, 1, *kr.switch_key(3))
    ctx.import_switch_key(0, 0, _cuda(rlk))
    ctx.import_switch_key(1, 1, _cuda(gk))
    g = synth.rng(15)
    a = np.stack([np.stack([synth.uniform_residues(g, p.q, p.N) for _ in range(2)]) for _ in range(2)])
    b = np.stack([np.stack([synth.uniform_residues(g, p.q, p.N) for _ in range(2)]) for _ in range(2)])
    A, B = ctx.import_coeffs(_cuda(a), 6, 1.0), ctx.import_coeffs(_cuda(b), 6, 1.0)
    got = _host(ctx.export_coeffs(ctx.rescale(ctx.mul_relin(A, B))))
    rot = _host(ctx.export_coeffs(ctx.rotate(A, 1)))
    for c in range(2):
        oa = oracle_mod.Ciphertext([a[c, 0], a[c, 1]], 6, 1.0)
        ob = oracle_mod.Ciphertext([b[c, 0], b[c, 1]], 6, 1.0)
        want = oracle_mod.rescale(p, oracle_mod.mul_relin(p, oa, ob, rlk))
        wr = oracle_mod.apply_galois(p, oa, kappa, gk)
        for k in range(2):
            assert np.array_equal(got[c, k], want.c[k]), (c, k)
            assert np.array_equal(rot[c, k], wr.c[k]), (c, k)
