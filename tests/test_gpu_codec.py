"""GPU parity of the batched encode / decode (P:140 ENCODE, P:143 DECODE).

Expected values come only from oracle/ (numpy FFT + Python big-integer CRT):
  * encode: every coefficient within +-1 of the oracle's rounded coefficient (reading A28),
    checked limb by limb -- the offset must be the same integer in every limb;
  * decode: slots within 2^-20 of the oracle's decode of the SAME residues (north star
    tolerance), and within 1e-12 relative for plaintexts whose coefficients reach 2^126
    (the exact mod-2^128 CRT lift, reading A33)."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1908_06972_b200 import synth  # noqa: E402

PRESETS = {"C1": (12, [30] * 3, 2.0 ** 30), "C4": (13, [60] + [40] * 4, 2.0 ** 40),
           "C2": (14, [40] * 8, 2.0 ** 40), "C3": (16, [40] * 30, 2.0 ** 40)}


@pytest.fixture(scope="module")
def ckks():
    from paper_1908_06972_b200 import ckks as m
    return m


_CTX = {}


def ctx_of(ckks, name):
    if name not in _CTX:
        log_n, bits, scale = PRESETS[name]
        _CTX[name] = ckks.Context(log_n, bits, 60, scale)
    return _CTX[name]


def _host(t) -> np.ndarray:
    return t.cpu().numpy().view(np.uint64)


def _offsets(got: np.ndarray, want: np.ndarray, q) -> np.ndarray:
    """got [l][N] residues, want [N] int64: the per-coefficient integer offset got - want,
    required to be one value in {-1, 0, 1} consistent across every limb."""
    offs = []
    for i, qi in enumerate(q):
        d = (got[i].astype(object) - want.astype(object)) % qi
        d = np.array([x if x <= qi // 2 else x - qi for x in d], dtype=np.int64)
        offs.append(d)
    offs = np.stack(offs)
    assert np.all(offs == offs[0]), "limbs disagree: not the residues of one integer"
    return offs[0]


@pytest.mark.parametrize("name,count,n_slots,cplx", [("C1", 3, 2048, False), ("C1", 2, 37, True),
                                                     ("C4", 4, 4096, True), ("C2", 2, 5000, False),
                                                     ("C3", 1, 32768, True)])
def test_encode_batch_vs_oracle(ckks, oracle_mod, name, count, n_slots, cplx):
    p = oracle_mod.preset(name)
    ctx = ctx_of(ckks, name)
    g = synth.rng(1000 + count + n_slots)
    zs = [synth.complex_slots(g, n_slots) if cplx else synth.real_slots(g, n_slots) for _ in range(count)]
    z = torch.from_numpy(np.stack(zs).astype(np.complex128)).cuda()
    lvl = p.L if name != "C2" else p.L - 3  # also a level below the top
    pt = ctx.encode_batch(z, level=lvl)
    assert pt.level == lvl and pt.scale == p.scale
    got = _host(ctx.export_coeffs(pt))
    n_off = 0
    for c in range(count):
        want = oracle_mod.encode_coeffs(zs[c], p.scale, p.log_n)
        off = _offsets(got[c, 0], want, p.q[:lvl])
        assert np.max(np.abs(off)) <= 1
        n_off += int(np.count_nonzero(off))
    assert n_off <= count * 4  # rounding-boundary disagreements only
    assert not ctx.encode_overflowed()


def test_encode_batch_empty_and_overflow(ckks, oracle_mod):
    p = oracle_mod.preset("C1")
    ctx = ctx_of(ckks, "C1")
    z = torch.zeros((2, 0), dtype=torch.complex128, device="cuda")
    pt = ctx.encode_batch(z)
    assert not np.any(_host(ctx.export_coeffs(pt)))  # zero vector -> zero polynomial
    big = torch.ones((1, p.slots), dtype=torch.complex128, device="cuda")
    ctx.encode_batch(big, scale=2.0 ** 70)  # all-ones vector = constant 2^70 > int64
    assert ctx.encode_overflowed()
    assert not ctx.encode_overflowed()  # sticky until read
    with pytest.raises(Exception):
        ctx.encode_batch(torch.zeros((1, p.slots + 1), dtype=torch.complex128, device="cuda"))


@pytest.mark.parametrize("name,count,n_slots", [("C1", 3, 2048), ("C4", 2, 100), ("C2", 2, 8192),
                                                ("C3", 1, 32768)])
def test_decode_batch_vs_oracle(ckks, oracle_mod, name, count, n_slots):
    """Decode of encoded vectors at every level from the top down to 1."""
    p = oracle_mod.preset(name)
    ctx = ctx_of(ckks, name)
    g = synth.rng(77 + count)
    for lvl in sorted({p.L, max(1, p.L // 2), 1}, reverse=True):
        zs = [synth.complex_slots(g, n_slots) for _ in range(count)]
        m = np.stack([oracle_mod.encode_coeffs(zc, p.scale, p.log_n) for zc in zs])
        res = np.stack([[oracle_mod.poly_from_signed(m[c], p.q[:lvl], p.log_n)] for c in range(count)])
        pt = ctx.import_coeffs(torch.from_numpy(res.view(np.int64)).cuda(), lvl, p.scale)
        out = ctx.decode_batch(pt, n_slots).cpu().numpy()
        for c in range(count):
            want = oracle_mod.decode(p, oracle_mod.Plaintext(res[c, 0], lvl, p.scale))[:n_slots]
            assert np.max(np.abs(out[c] - want)) <= 2.0 ** -20, (lvl, c)
            assert np.max(np.abs(out[c] - zs[c])) <= p.N * 2.0 ** (-math.log2(p.scale)) * 4


def test_decode_batch_wide_coefficients(ckks, oracle_mod):
    """Coefficients up to +-2^126 (multi-word CRT lift, reading A33) at C2 (Q ~ 2^320)."""
    p = oracle_mod.preset("C2")
    ctx = ctx_of(ckks, "C2")
    g = synth.rng(5)
    n = p.N
    mag = g.integers(0, 2 ** 62, size=n, dtype=np.int64)
    sign = g.integers(0, 2, size=n)
    ints = [(-1 if s else 1) * ((int(x) << 64) + int(y)) for x, y, s in
            zip(mag, g.integers(0, 2 ** 63, size=n, dtype=np.int64), sign)]
    ints[0], ints[1], ints[2] = 2 ** 126 - 1, -(2 ** 126 - 1), 0
    Q = math.prod(p.q)
    res = np.array([[x % qi for x in ints] for qi in p.q], dtype=np.uint64)
    pt = ctx.import_coeffs(torch.from_numpy(res[None, None].view(np.int64)).cuda(), p.L, 2.0 ** 100)
    out = ctx.decode_batch(pt).cpu().numpy()[0]
    want = oracle_mod.decode_coeffs(np.array([float(x) for x in ints]), 2.0 ** 100, p.log_n)
    assert oracle_mod.centered(oracle_mod.crt_int(res, p.q), Q) == ints  # the input really is those integers
    assert np.max(np.abs(out - want)) <= 1e-12 * np.max(np.abs(want))


def test_codec_roundtrip_through_encryption(ckks, oracle_mod):
    """encode_batch -> encrypt -> HMult -> rescale -> decrypt -> decode_batch ~ z^2."""
    p = oracle_mod.preset("C1")
    ctx = ctx_of(ckks, "C1")
    kr = synth.KeyRandomness(3, p.log_n, p.q, p.P)

    def dev(a):
        a = np.ascontiguousarray(a)
        return torch.from_numpy(a.view(np.int64) if a.dtype == np.uint64 else a).cuda()

    ctx.set_secret(dev(kr.s))
    ctx.keygen_public(dev(kr.pk_a), dev(kr.pk_e))
    a, e = kr.switch_key(1)
    ctx.keygen_relin(dev(a), dev(e))
    g = synth.rng(11)
    count = 3
    zs = np.stack([synth.real_slots(g, p.slots) for _ in range(count)])
    pt = ctx.encode_batch(torch.from_numpy(zs.astype(np.complex128)).cuda())
    us, e0s, e1s = zip(*[kr.enc(100 + c) for c in range(count)])
    ct = ctx.encrypt(pt, dev(np.stack(us)), dev(np.stack(e0s)), dev(np.stack(e1s)))
    sq = ctx.rescale(ctx.mul_relin(ct, ct))
    dec = ctx.decrypt(sq)
    out = ctx.decode_batch(dec).cpu().numpy()
    want = oracle_mod.decode(p, oracle_mod.Plaintext(_host(ctx.export_coeffs(dec))[0, 0], dec.level, dec.scale))
    assert np.max(np.abs(out[0] - want)) <= 2.0 ** -20
    assert np.max(np.abs(out - zs ** 2)) < 1e-2  # C1: Delta = 2^30, N = 2^12 -> ~1e-3 noise
