"""ckks_mul_relin_rescale: the key switch's ModDown and the RESCALE as one floor by P q_{l-1}
(reading A7).  Must be bit-identical to the oracle's mul_relin followed by rescale (Eq. 1) at
every ring, level and batch, including the 60-bit q_0 (C4) and the full C3 size; the hybrid
(alpha > 1) path runs the two steps in sequence."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1908_06972_b200 import synth  # noqa: E402


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).cuda()


def _host(t):
    return t.cpu().numpy().view(np.uint64)


def _rand(p, cnt, level, seed):
    g = synth.rng(seed)
    return np.stack([np.stack([synth.uniform_residues(g, p.q[:level], p.N) for _ in range(2)]) for _ in range(cnt)])


@pytest.mark.parametrize("log_n,bits,levels,count", [(12, [30] * 3, (3, 2), 3), (13, [60] + [40] * 4, (5, 3, 2), 4),
                                                     (14, [40] * 8, (8, 5), 2), (16, [40] * 30, (30,), 1)])
def test_mul_relin_rescale_vs_oracle(oracle_mod, log_n, bits, levels, count):
    from paper_1908_06972_b200 import ckks
    qs, sp = oracle_mod.prime_chain(log_n, bits)
    p = oracle_mod.Params(log_n, qs, sp[0], 2.0 ** 40)
    ctx = ckks.Context(log_n, bits, 60, 2.0 ** 40)
    assert ctx.q == p.q
    g = synth.rng(77 + log_n)
    ext = list(p.ext_mods())
    rlk = np.stack([np.stack([synth.uniform_residues(g, ext, p.N) for _ in range(2)]) for _ in range(p.L)])
    ctx.import_switch_key(0, 0, _cuda(rlk))
    for level in levels:
        a, b = _rand(p, count, level, 1 + level), _rand(p, count, level, 50 + level)
        A, B = ctx.import_coeffs(_cuda(a), level, 2.0 ** 40), ctx.import_coeffs(_cuda(b), level, 2.0 ** 40)
        out = ctx.mul_relin_rescale(A, B)
        assert out.level == level - 1 and out.scale == 2.0 ** 80 / float(p.q[level - 1])
        got = _host(ctx.export_coeffs(out))
        seq = _host(ctx.export_coeffs(ctx.rescale(ctx.mul_relin(A, B))))
        assert np.array_equal(got, seq)
        for c in range(count):
            want = oracle_mod.rescale(p, oracle_mod.mul_relin(p, oracle_mod.Ciphertext([a[c, 0], a[c, 1]], level, 1.0),
                                                               oracle_mod.Ciphertext([b[c, 0], b[c, 1]], level, 1.0),
                                                               rlk))
            for k in range(2):
                assert np.array_equal(got[c, k], want.c[k]), (level, c, k)
    A1 = ctx.import_coeffs(_cuda(_rand(p, 1, 1, 9)), 1, 1.0)
    with pytest.raises(ckks.CkksError):
        ctx.mul_relin_rescale(A1, A1)
    ctx.close()


def test_mul_relin_rescale_hybrid_falls_back(oracle_mod):
    from paper_1908_06972_b200 import ckks
    p = oracle_mod.toy_params(12, [30] * 6, 60, alpha=3, n_special=2)
    ctx = ckks.Context(12, [30] * 6, 60, 2.0 ** 20, n_special=2, digit_limbs=3)
    g = synth.rng(5)
    rlk = np.stack([np.stack([synth.uniform_residues(g, list(p.ext_mods()), p.N) for _ in range(2)])
                    for _ in range(p.dnum)])
    ctx.import_switch_key(0, 0, _cuda(rlk))
    a, b = _rand(p, 2, 6, 3), _rand(p, 2, 6, 4)
    A, B = ctx.import_coeffs(_cuda(a), 6, 1.0), ctx.import_coeffs(_cuda(b), 6, 1.0)
    got = _host(ctx.export_coeffs(ctx.mul_relin_rescale(A, B)))
    for c in range(2):
        want = oracle_mod.rescale(p, oracle_mod.mul_relin(p, oracle_mod.Ciphertext([a[c, 0], a[c, 1]], 6, 1.0),
                                                           oracle_mod.Ciphertext([b[c, 0], b[c, 1]], 6, 1.0), rlk))
        assert np.array_equal(got[c, 0], want.c[0]) and np.array_equal(got[c, 1], want.c[1])
    ctx.close()
