"""GPU parity of the alternative kernel paths at the PrivFT inference ring (SURVEY C4,
N = 2^13): every variant must be bit-identical to the oracle.

* CKKS_SPLIT_CLASSES=1: single-class (FP64-only / integer-only) column launches at C4 (auto
  mode keeps them mixed there);
* CKKS_INV_MODUP=0/1: the digits' INTT column phase fused with the ModUp column phases off /
  forced on (auto: on when the launch has >= 16 CTAs per SM);
* CKKS_INV_BCAST=0/1: the ModDown / rescale source limb's INTT column phase fused with the
  broadcast column phases off / forced on;
* CKKS_DUAL_STREAM=0: integer- and FP64-class inner products on one stream (default: two);
* CKKS_KSMAC_INT=1: the integer key-switch classes on the original double-buffered body;
* CKKS_NTT_F64=0: integer-pipe NTT for every prime (FP64 mode off) -- read at context creation;
* CKKS_CHUNKDOT_TC=0: CUDA-core chunk-dot instead of the tensor-core one (model creation)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1908_06972_b200 import synth  # noqa: E402


def _cuda(a):
    a = np.ascontiguousarray(a)
    return torch.from_numpy(a.view(np.int64) if a.dtype == np.uint64 else a).cuda()


def _host(t):
    return t.cpu().numpy().view(np.uint64)


@pytest.fixture(scope="module")
def c4(oracle_mod):
    p = oracle_mod.preset("C4")
    kr = synth.KeyRandomness(13, p.log_n, p.q, p.P)
    rlk = oracle_mod.keygen_relin(p, kr.s, *kr.switch_key(0))
    gk = {}
    for st in (1, 2):
        kappa, key = oracle_mod.keygen_galois(p, kr.s, st, *kr.switch_key(100 + st))
        gk[kappa] = (st, key)
    return dict(p=p, rlk=rlk, gk=gk)


def _ctx(ckks, c4):
    p = c4["p"]
    ctx = ckks.Context(p.log_n, [60, 40, 40, 40, 40], 60, p.scale)
    assert ctx.q == p.q
    ctx.import_switch_key(0, 0, _cuda(c4["rlk"]))
    for kappa, (st, key) in c4["gk"].items():
        ctx.import_switch_key(1, st, _cuda(key))
    return ctx


def _rand(p, cnt, level, seed):
    g = synth.rng(seed)
    return np.stack([np.stack([synth.uniform_residues(g, p.q[:level], p.N) for _ in range(2)]) for _ in range(cnt)])


@pytest.mark.parametrize("env", [{"CKKS_NTT_F64": "0"},
                                 {"CKKS_SPLIT_CLASSES": "1"}, {"CKKS_KSMAC_INT": "1"},
                                 {"CKKS_INV_MODUP": "0"},
                                 {"CKKS_INV_MODUP": "1"}, {"CKKS_INV_BCAST": "0"}, {"CKKS_INV_BCAST": "1"},
                                 {"CKKS_DUAL_STREAM": "0"}, {}])
@pytest.mark.parametrize("level", [5, 4])
def test_keyswitch_variants_bit_exact(oracle_mod, c4, monkeypatch, env, level):
    from paper_1908_06972_b200 import ckks
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    p = c4["p"]
    ctx = _ctx(ckks, c4)
    a, b = _rand(p, 2, level, 7 + level), _rand(p, 2, level, 9 + level)
    A, B = ctx.import_coeffs(_cuda(a), level, 1.0), ctx.import_coeffs(_cuda(b), level, 1.0)
    got = _host(ctx.export_coeffs(ctx.mul_relin(A, B)))
    rot = _host(ctx.export_coeffs(ctx.rotate(A, 2)))
    gk = {k: v[1] for k, v in c4["gk"].items()}
    for c in range(2):
        ca = oracle_mod.Ciphertext([a[c, 0], a[c, 1]], level, 1.0)
        want = oracle_mod.mul_relin(p, ca, oracle_mod.Ciphertext([b[c, 0], b[c, 1]], level, 1.0), c4["rlk"])
        wr = oracle_mod.rotate(p, ca, 2, gk)
        for k in range(2):
            assert np.array_equal(got[c, k], want.c[k]), (env, c, k)
            assert np.array_equal(rot[c, k], wr.c[k]), (env, c, k)
    ctx.close()


@pytest.mark.parametrize("tc", ["1", "0"])
def test_chunkdot_variants_bit_exact(oracle_mod, c4, monkeypatch, tc):
    """v.H chunk-dot at N = 2^13 (tensor-core byte-plane path vs CUDA-core path) vs the
    oracle's sum of HMULPLAIN + HADD, on uniform residues, B = 3 queries, K = 5, n = 11."""
    from paper_1908_06972_b200 import ckks
    monkeypatch.setenv("CKKS_CHUNKDOT_TC", tc)
    p = c4["p"]
    ctx = _ctx(ckks, c4)
    B, K, n, L = 3, 5, 11, p.L
    g = synth.rng(31)
    bag = np.stack([np.stack([synth.uniform_residues(g, p.q, p.N) for _ in range(2)]) for _ in range(B * K)])
    H = np.stack([synth.uniform_residues(g, p.q, p.N)[None] for _ in range(n * K)])
    O = np.stack([synth.uniform_residues(g, p.q[:L - 2], p.N)[None] for _ in range(n)])
    Hd = ctx.import_coeffs(_cuda(H), L, p.scale)
    Od = ctx.import_coeffs(_cuda(O), L - 2, p.scale)
    model = ctx.privft_model_wrap(Hd, Od, K * p.slots, n, 2)
    got = _host(ctx.export_coeffs(ctx.privft_chunkdot(model, ctx.import_coeffs(_cuda(bag), L, p.scale))))
    for b in range(B):
        for j in range(n):
            acc = None
            for k in range(K):
                x = oracle_mod.mul_plain(p, oracle_mod.Ciphertext(list(bag[b * K + k]), L, 1.0),
                                         oracle_mod.Plaintext(H[j * K + k, 0], L, 1.0))
                acc = x if acc is None else oracle_mod.add(p, acc, x)
            assert np.array_equal(got[b * n + j, 0], acc.c[0]) and np.array_equal(got[b * n + j, 1], acc.c[1])
    ctx.close()


def test_digit_split_keyswitch_bit_exact(oracle_mod, monkeypatch):
    """The digit-split inner product (a launch too small to fill the GPU runs its digit loop
    over several CTA rows and sums canonical partials): one ciphertext at N = 2^14, l = 12,
    so the special-prime target (integer class) and every FP64 target launch split."""
    from paper_1908_06972_b200 import ckks
    log_n, L = 14, 12
    qs, sp = oracle_mod.prime_chain(log_n, [40] * L)
    p = oracle_mod.Params(log_n, qs, sp[0], 2.0 ** 30)
    ctx = ckks.Context(log_n, [40] * L, 60, p.scale)
    assert ctx.q == p.q
    kr = synth.KeyRandomness(5, p.log_n, p.q, p.P)
    rlk = oracle_mod.keygen_relin(p, kr.s, *kr.switch_key(0))
    ctx.import_switch_key(0, 0, _cuda(rlk))
    a, b = _rand(p, 1, L, 3), _rand(p, 1, L, 4)
    A, B = ctx.import_coeffs(_cuda(a), L, 1.0), ctx.import_coeffs(_cuda(b), L, 1.0)
    ctx.profile(True)
    got = _host(ctx.export_coeffs(ctx.mul_relin(A, B)))
    ctx.profile(False)
    assert "ks_split_sum" in ctx.profile_read()
    want = oracle_mod.mul_relin(p, oracle_mod.Ciphertext([a[0, 0], a[0, 1]], L, 1.0),
                                oracle_mod.Ciphertext([b[0, 0], b[0, 1]], L, 1.0), rlk)
    assert np.array_equal(got[0, 0], want.c[0]) and np.array_equal(got[0, 1], want.c[1])
    ctx.close()


@pytest.mark.parametrize("log_n,L", [(12, 4), (14, 8), (15, 6), (16, 5)])
def test_fused_column_kernels_every_ring(oracle_mod, monkeypatch, log_n, L):
    """The fused INTT+ModUp and INTT+broadcast column kernels forced on and off at every
    column/row geometry (they switch on automatically only for large batches at N = 2^13):
    HMult+relin+rescale and rotate(2) bit-exact against the oracle either way."""
    from paper_1908_06972_b200 import ckks
    bits = [60] + [40] * (L - 1)
    qs, sp = oracle_mod.prime_chain(log_n, bits)
    p = oracle_mod.Params(log_n, qs, sp[0], 2.0 ** 40)
    g = synth.rng(100 + log_n)
    ext = list(p.ext_mods())
    key = lambda: np.stack([np.stack([synth.uniform_residues(g, ext, p.N) for _ in range(2)]) for _ in range(L)])
    rlk, gk = key(), key()
    kappa = oracle_mod.galois_elt(p, 2)
    a, b = _rand(p, 3, L, 1), _rand(p, 3, L, 2)
    want_m, want_r = [], []
    for c in range(3):
        oa = oracle_mod.Ciphertext([a[c, 0], a[c, 1]], L, 1.0)
        ob = oracle_mod.Ciphertext([b[c, 0], b[c, 1]], L, 1.0)
        want_m.append(oracle_mod.rescale(p, oracle_mod.mul_relin(p, oa, ob, rlk)))
        want_r.append(oracle_mod.rotate(p, oa, 2, {kappa: gk}))
    for forced in ("0", "1"):
        monkeypatch.setenv("CKKS_INV_MODUP", forced)
        monkeypatch.setenv("CKKS_INV_BCAST", forced)
        ctx = ckks.Context(log_n, bits, 60, 2.0 ** 40)
        assert ctx.q == p.q and ctx.P == p.P
        ctx.import_switch_key(0, 0, _cuda(rlk))
        ctx.import_switch_key(1, 2, _cuda(gk))
        A, B = ctx.import_coeffs(_cuda(a), L, 1.0), ctx.import_coeffs(_cuda(b), L, 1.0)
        got_m = _host(ctx.export_coeffs(ctx.rescale(ctx.mul_relin(A, B))))
        got_r = _host(ctx.export_coeffs(ctx.rotate(A, 2)))
        for c in range(3):
            for k in range(2):
                assert np.array_equal(got_m[c, k], want_m[c].c[k]), (forced, c, k)
                assert np.array_equal(got_r[c, k], want_r[c].c[k]), (forced, c, k)
        ctx.close()


@pytest.mark.parametrize("log_n,L,count", [(12, 3, 3), (13, 5, 7), (14, 8, 2), (15, 6, 1), (16, 5, 1)])
def test_cluster_keyswitch_vs_oracle(oracle_mod, monkeypatch, log_n, L, count):
    """The thread-block-cluster key switch (ks_cluster.cu, CKKS_KS_CLUSTER=1): every cluster
    size (1, 2, 4, 8, 16 CTAs), 60-bit q_0 and P on the two-kernel path beside it, segments cut
    between clusters; HMult+relin+rescale and rotate(3) bit-exact against the oracle."""
    from paper_1908_06972_b200 import ckks
    monkeypatch.setenv("CKKS_KS_CLUSTER", "1")
    bits = [60] + [40] * (L - 1)
    qs, sp = oracle_mod.prime_chain(log_n, bits)
    p = oracle_mod.Params(log_n, qs, sp[0], 2.0 ** 40)
    g = synth.rng(200 + log_n)
    ext = list(p.ext_mods())
    key = lambda: np.stack([np.stack([synth.uniform_residues(g, ext, p.N) for _ in range(2)]) for _ in range(L)])
    rlk = key()
    gks = {st: key() for st in oracle_mod.rotation_steps(p, 3)}
    a, b = _rand(p, count, L, 3), _rand(p, count, L, 4)
    ctx = ckks.Context(log_n, bits, 60, 2.0 ** 40)
    assert ctx.q == p.q and ctx.P == p.P
    ctx.import_switch_key(0, 0, _cuda(rlk))
    for st, k in gks.items():
        ctx.import_switch_key(1, st, _cuda(k))
    A, B = ctx.import_coeffs(_cuda(a), L, 1.0), ctx.import_coeffs(_cuda(b), L, 1.0)
    ctx.profile(True)
    got_m = _host(ctx.export_coeffs(ctx.rescale(ctx.mul_relin(A, B))))
    got_r = _host(ctx.export_coeffs(ctx.rotate(A, 3)))
    ctx.profile(False)
    assert "ks_cluster" in ctx.profile_read()
    gk = {oracle_mod.galois_elt(p, st): k for st, k in gks.items()}
    for c in range(count):
        oa = oracle_mod.Ciphertext([a[c, 0], a[c, 1]], L, 1.0)
        ob = oracle_mod.Ciphertext([b[c, 0], b[c, 1]], L, 1.0)
        wm = oracle_mod.rescale(p, oracle_mod.mul_relin(p, oa, ob, rlk))
        wr = oracle_mod.rotate(p, oa, 3, gk)
        for k in range(2):
            assert np.array_equal(got_m[c, k], wm.c[k]), (c, k)
            assert np.array_equal(got_r[c, k], wr.c[k]), (c, k)
    ctx.close()
