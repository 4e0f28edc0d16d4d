"""Persistence / client-server boundary ("the client ... sends the encrypted
input", P:465 the 123-ciphertext request; S:429 the server never holds s):

* ckks_export / ckks_import: host bytes in coefficient form round-trip bit-exactly, across
  contexts of the same parameters, and are refused for another chain, a corrupt header, a
  truncated buffer or a residue >= q_i;
* ckks_export_keys: the serialised relinearisation, Galois and public keys equal the ORACLE's
  keygen (coefficient form) for the same randomness, with and without the cluster key switch's
  MAC layout; ckks_import_keys on a context without the secret reproduces the oracle's HMult and
  rotation."""
import struct

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


def test_export_import_roundtrip_and_rejections(oracle_mod):
    from paper_1908_06972_b200 import ckks
    p = oracle_mod.preset("C4")
    ctx = ckks.Context(13, [60, 40, 40, 40, 40], 60, 2.0 ** 40)
    a = _rand(p, 3, 4, 1)
    A = ctx.import_coeffs(_cuda(a), 4, 1234.5)
    blob = ctx.export(A)
    magic, ver, log_n, cnt, npl, lev, zero, scale = struct.unpack_from("<8s6Id", blob, 0)
    assert (magic, ver, log_n, cnt, npl, lev, scale) == (b"CKKSBUF1", 1, 13, 3, 2, 4, 1234.5)
    assert np.array_equal(np.frombuffer(blob[64:], dtype=np.uint64).reshape(a.shape), a)  # coefficient form
    B = ctx.import_bytes(blob)
    assert (B.level, B.scale, B.count) == (4, 1234.5, 3) and torch.equal(B.t, A.t)
    other = ckks.Context(13, [60, 40, 40, 40, 40], 60, 2.0 ** 40)  # a fresh context, same parameters
    assert torch.equal(other.import_bytes(blob).t, A.t)
    c1 = ckks.Context(13, [40] * 5, 60, 2.0 ** 40)  # another chain
    with pytest.raises(ckks.CkksError):
        c1.import_bytes(blob)
    bad = bytearray(blob)
    bad[0:8] = b"XXXXXXXX"
    with pytest.raises(ckks.CkksError):
        ctx.import_bytes(bytes(bad))
    with pytest.raises(ckks.CkksError):
        ctx.import_bytes(blob[:-8])
    bad = bytearray(blob)
    bad[64:72] = struct.pack("<Q", p.q[0])  # residue == q_0: not canonical
    with pytest.raises(ckks.CkksError):
        ctx.import_bytes(bytes(bad))
    for x in (ctx, other, c1):
        x.close()


@pytest.mark.parametrize("cluster", ["0", "1"])
def test_export_keys_equal_oracle_keygen_and_serve(oracle_mod, monkeypatch, cluster):
    from paper_1908_06972_b200 import ckks
    monkeypatch.setenv("CKKS_KS_CLUSTER", cluster)
    p = oracle_mod.preset("C4")
    kr = synth.KeyRandomness(21, p.log_n, p.q, p.P)
    ar, er = kr.switch_key(0)
    ag, eg = kr.switch_key(1)
    client = ckks.Context(13, [60, 40, 40, 40, 40], 60, 2.0 ** 40)
    client.set_secret(_cuda(kr.s))
    client.keygen_public(_cuda(kr.pk_a), _cuda(kr.pk_e))
    client.keygen_relin(_cuda(ar), _cuda(er))
    client.keygen_galois(2, _cuda(ag), _cuda(eg))
    blob = client.export_keys()
    magic, ver, log_n, L, K, alpha, n_keys, chain = struct.unpack_from("<8s6IQ", blob, 0)
    assert (magic, log_n, L, K, alpha, n_keys) == (b"CKKSKEY1", 13, 5, 1, 1, 3)
    want_pk = oracle_mod.keygen_public(p, kr.s, kr.pk_a, kr.pk_e)
    want_rlk = oracle_mod.keygen_relin(p, kr.s, ar, er)
    kappa, want_gk = oracle_mod.keygen_galois(p, kr.s, 2, ag, eg)
    off, seen = 64, {}
    kw, pw = want_rlk.size, 2 * p.L * p.N
    for _ in range(n_keys):
        kind, _z, kap = struct.unpack_from("<IIQ", blob, off)
        off += 16
        w = pw if kind == 2 else kw
        seen[(kind, kap)] = np.frombuffer(blob[off:off + 8 * w], dtype=np.uint64)
        off += 8 * w
    assert off == len(blob)
    assert np.array_equal(seen[(2, 0)].reshape(2, p.L, p.N), np.stack(want_pk))
    assert np.array_equal(seen[(0, 0)].reshape(want_rlk.shape), want_rlk)
    assert np.array_equal(seen[(1, kappa)].reshape(want_gk.shape), want_gk)
    # the server: no secret, keys from the bytes only
    server = ckks.Context(13, [60, 40, 40, 40, 40], 60, 2.0 ** 40)
    server.import_keys(blob)
    a, b = _rand(p, 2, 5, 5), _rand(p, 2, 5, 6)
    A, B = server.import_coeffs(_cuda(a), 5, 1.0), server.import_coeffs(_cuda(b), 5, 1.0)
    got_m = _host(server.export_coeffs(server.mul_relin(A, B)))
    got_r = _host(server.export_coeffs(server.rotate(A, 2)))
    for c in range(2):
        oa = oracle_mod.Ciphertext([a[c, 0], a[c, 1]], 5, 1.0)
        ob = oracle_mod.Ciphertext([b[c, 0], b[c, 1]], 5, 1.0)
        wm = oracle_mod.mul_relin(p, oa, ob, want_rlk)
        wr = oracle_mod.apply_galois(p, oa, kappa, want_gk)
        for k in range(2):
            assert np.array_equal(got_m[c, k], wm.c[k]) and np.array_equal(got_r[c, k], wr.c[k])
    with pytest.raises(ckks.CkksError):  # keys of another parameter set
        ckks.Context(13, [40] * 5, 60, 2.0 ** 40).import_keys(blob)
    client.close()
    server.close()
