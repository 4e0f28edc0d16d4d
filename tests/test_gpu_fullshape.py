"""GPU parity at the shapes the bench and the north star name, element by element against
the oracle (VERDICT r1 "next round" item 1):

* the v.H chunk-dot with K = 300 chunks and a 60-bit q_0, NTT-domain residues near q - 1
  (the 128-bit accumulator bound: K (q-1)^2 wraps 2^128 for K >= 256 at 60 bits), on the
  tensor-core and the CUDA-core paths;
* rotation at C3 (N = 2^16, l = 30): rotate(1), rotate(-1) and the two-digit NAF step 3 =
  4 - 1 (reading A10); the HHW step 21845 (NAF weight 8, Table 2) with
  CKKS_RUN_SLOW=1;
* hybrid key switching at the bench's C3 shape alpha = 10, K = 7 (row f2): HMult+relin+
  rescale;
* privft_infer at the bench's exact shape (C4, m = 500,000 -> K = 123, n = 300, c = 4, B = 32,
  poly softmax, default chunking): 64 sampled (b, j) chunk-dot outputs and one full query's
  scores bit-exact.

Random uniform residues stand in for keys, plaintexts and ciphertexts: every step checked
here is exact ring arithmetic, defined on any residues."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1908_06972_b200 import synth  # noqa: E402

NPROC = os.cpu_count() or 1


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).cuda()


def _host(t):
    return t.cpu().numpy().view(np.uint64)


def _uni_key(g, p, dnum, ext):
    return np.stack([np.stack([synth.uniform_residues(g, ext, p.N) for _ in range(2)]) for _ in range(dnum)])


# ---------------------------------------------------------------- chunk-dot, K = 300 --
@pytest.mark.parametrize("tc,K,B,sb", [("1", 300, 2, ""), ("0", 300, 2, ""), ("1", 20, 5, "2")])
def test_chunkdot_k300_60bit_near_q(oracle_mod, monkeypatch, tc, K, B, sb):
    """v.H chunk-dot with every operand near q (128-bit accumulator folding at K = 300 chunks, 60-bit
    q_0), tensor-core and CUDA-core paths; and the tensor-core path in sub-batches of 2 queries
    with a ragged last one (how batches too large for one shared-memory tile run)."""
    from paper_1908_06972_b200 import ckks
    monkeypatch.setenv("CKKS_CHUNKDOT_TC", tc)
    if sb:
        monkeypatch.setenv("CKKS_CHUNKDOT_SB", sb)
    log_n, bits = 10, [60, 40, 40, 40]  # the packed model needs L >= 4
    qs, sp = oracle_mod.prime_chain(log_n, bits)
    p = oracle_mod.Params(log_n, qs, sp[0], 2.0 ** 40)
    ctx = ckks.Context(log_n, bits, 60, 2.0 ** 40)
    assert ctx.q == p.q and p.q[0] > (1 << 59)
    t, n = p.slots, 3
    m = K * t
    g = synth.rng(300)

    def near_top():  # coefficient form whose NTT-domain values all lie in [q - 2^12, q - 1]
        return np.stack([oracle_mod.ntt_inv(q - 1 - g.integers(0, 1 << 12, size=p.N, dtype=np.uint64), log_n, q)
                         for q in p.q])

    H = np.stack([near_top() for _ in range(n * K)])[:, None]            # [n K][1][L][N]
    O = np.stack([synth.uniform_residues(g, p.q[:2], p.N) for _ in range(n)])[:, None]
    bag = np.stack([np.stack([near_top(), near_top()]) for _ in range(B * K)])  # [B K][2][L][N]
    model = ctx.privft_model_wrap(ctx.import_coeffs(_cuda(H), 4, p.scale), ctx.import_coeffs(_cuda(O), 2, p.scale),
                                  m, n, 2)
    got = _host(ctx.export_coeffs(ctx.privft_chunkdot(model, ctx.import_coeffs(_cuda(bag), 4, p.scale))))
    for b in range(B):
        for j in range(n):
            want = [None, None]
            for k in range(K):
                for poly in range(2):
                    prod = oracle_mod.poly_mul(bag[b * K + k, poly], H[j * K + k, 0], p.q, log_n)
                    want[poly] = prod if want[poly] is None else oracle_mod.poly_add(want[poly], prod, p.q, log_n)
            for poly in range(2):
                assert np.array_equal(got[b * n + j, poly], want[poly]), (b, j, poly)


# ----------------------------------------------------------------------- C3 rotations --
@pytest.fixture(scope="module")
def c3(oracle_mod):
    from paper_1908_06972_b200 import ckks
    p = oracle_mod.preset("C3")
    ctx = ckks.Context(16, [40] * 30, 60, 2.0 ** 40)
    assert ctx.q == p.q and ctx.P == p.P
    g = synth.rng(1616)
    a = np.stack([synth.uniform_residues(g, p.q, p.N) for _ in range(2)])[None]
    yield dict(p=p, ctx=ctx, g=g, a=a, A=ctx.import_coeffs(_cuda(a), 30, p.scale), keys={})
    ctx.close()


def _c3_keys(oracle_mod, w, steps):
    p, ctx = w["p"], w["ctx"]
    for st in steps:
        kappa = oracle_mod.galois_elt(p, st)
        if kappa not in w["keys"]:
            key = _uni_key(w["g"], p, p.L, list(p.ext_mods()))
            ctx.import_switch_key(1, st, _cuda(key))
            w["keys"][kappa] = key
    return w["keys"]


@pytest.mark.parametrize("steps", [1, -1, 3])
def test_c3_rotate_vs_oracle(oracle_mod, c3, steps):
    p, ctx = c3["p"], c3["ctx"]
    gk = _c3_keys(oracle_mod, c3, oracle_mod.rotation_steps(p, steps))
    got = _host(ctx.export_coeffs(ctx.rotate(c3["A"], steps)))[0]
    want = oracle_mod.rotate(p, oracle_mod.Ciphertext([c3["a"][0, 0], c3["a"][0, 1]], 30, p.scale), steps, gk)
    assert np.array_equal(got[0], want.c[0]) and np.array_equal(got[1], want.c[1])


def test_c3_rotate_hhw_21845_vs_oracle(oracle_mod, c3):
    """Table 2's high-Hamming-weight rotation at N = 2^16 (NAF weight 8: eight key switches with
    8 C3 Galois keys, ~8 GB) bit-exact against the oracle (~30 s on one B200)."""
    p, ctx = c3["p"], c3["ctx"]
    assert len(oracle_mod.rotation_steps(p, 21845)) == 8  # NAF weight 8 (P14)
    gk = _c3_keys(oracle_mod, c3, oracle_mod.rotation_steps(p, 21845))
    got = _host(ctx.export_coeffs(ctx.rotate(c3["A"], 21845)))[0]
    want = oracle_mod.rotate(p, oracle_mod.Ciphertext([c3["a"][0, 0], c3["a"][0, 1]], 30, p.scale), 21845, gk)
    assert np.array_equal(got[0], want.c[0]) and np.array_equal(got[1], want.c[1])


# -------------------------------------------------------------- hybrid alpha=10, K=7 --
@pytest.mark.parametrize("K,sp_bits", [(7, 60), (10, 41), (10, 40)])
def test_c3_hybrid_a10_k7_hmult_vs_oracle(oracle_mod, K, sp_bits):
    """C3 hybrid HMult+relin+rescale, two calls and the fused one-call tail, at the bench's two
    special-prime sets: K = 7 x 60-bit (integer-pipe special slots) and K = 10 x 41-bit (FP64)."""
    from paper_1908_06972_b200 import ckks
    p = oracle_mod.toy_params(16, [40] * 30, sp_bits, scale=2.0 ** 40, alpha=10, n_special=K)
    ctx = ckks.Context(16, [40] * 30, sp_bits, 2.0 ** 40, n_special=K, digit_limbs=10)
    assert ctx.q == p.q and ctx.special == p.special and p.dnum == 3
    g = synth.rng(1007)
    rlk = _uni_key(g, p, p.dnum, list(p.ext_mods()))
    ctx.import_switch_key(0, 0, _cuda(rlk))
    a = np.stack([synth.uniform_residues(g, p.q, p.N) for _ in range(2)])[None]
    b = np.stack([synth.uniform_residues(g, p.q, p.N) for _ in range(2)])[None]
    A, B = ctx.import_coeffs(_cuda(a), 30, p.scale), ctx.import_coeffs(_cuda(b), 30, p.scale)
    got = _host(ctx.export_coeffs(ctx.rescale(ctx.mul_relin(A, B))))[0]
    got_f = _host(ctx.export_coeffs(ctx.mul_relin_rescale(A, B)))[0]  # fused ModDown + rescale tail
    want = oracle_mod.rescale(p, oracle_mod.mul_relin(p, oracle_mod.Ciphertext([a[0, 0], a[0, 1]], 30, p.scale),
                                                       oracle_mod.Ciphertext([b[0, 0], b[0, 1]], 30, p.scale), rlk))
    assert np.array_equal(got[0], want.c[0]) and np.array_equal(got[1], want.c[1])
    assert np.array_equal(got_f[0], want.c[0]) and np.array_equal(got_f[1], want.c[1])
    # hybrid rotation at N = 2^16 (the INTT row phase with the Galois gather, then the fused
    # ModUp column kernel / inner product / ModDown), steps 1 and -1
    for st in (1, -1):
        kappa = oracle_mod.galois_elt(p, st)
        gk = _uni_key(g, p, p.dnum, list(p.ext_mods()))
        ctx.import_switch_key(1, st, _cuda(gk))
        got_r = _host(ctx.export_coeffs(ctx.rotate(A, st)))[0]
        want_r = oracle_mod.apply_galois(p, oracle_mod.Ciphertext([a[0, 0], a[0, 1]], 30, p.scale), kappa, gk)
        assert np.array_equal(got_r[0], want_r.c[0]) and np.array_equal(got_r[1], want_r.c[1]), st
    ctx.close()


# ------------------------------------------------------------- PrivFT at bench shape --
M_, N_COLS, CLS, BATCH = 500000, 300, 4, 32


class _HCols:
    """H plaintexts generated per embedding column j from a seeded stream (12 GB in total:
    never held on the host at once).  H[j][k] = P^H_{j,k} (A17 layout, random residues)."""

    def __init__(self, oracle_mod, p, K):
        self.o, self.p, self.K = oracle_mod, p, K

    def raw(self, j):
        g = synth.rng(50000 + j)
        return np.stack([synth.uniform_residues(g, self.p.q, self.p.N) for _ in range(self.K)])

    def __getitem__(self, j):
        return [self.o.Plaintext(x, self.p.L, self.p.scale) for x in self.raw(j)]

    def __len__(self):
        return N_COLS


def _bag_raw(p, K, b):
    g = synth.rng(60000 + b)
    return np.stack([np.stack([synth.uniform_residues(g, p.q, p.N) for _ in range(2)]) for _ in range(K)])


_SAMPLE_CTX = None


def _chunkdot_sample(bj):
    o, p, K, Hc = _SAMPLE_CTX
    b, j = bj
    bag, H = _bag_raw(p, K, b), Hc[j]
    acc = None
    for k in range(K):
        t = o.mul_plain(p, o.Ciphertext([bag[k, 0], bag[k, 1]], p.L, p.scale), H[k])
        acc = t if acc is None else o.add(p, acc, t)
    return acc.c[0], acc.c[1]


def test_privft_bench_shape_vs_oracle(oracle_mod):
    import multiprocessing as mp
    from paper_1908_06972_b200 import ckks
    global _SAMPLE_CTX
    p = oracle_mod.preset("C4")
    ctx = ckks.Context(13, [60, 40, 40, 40, 40], 60, 2.0 ** 40)
    assert ctx.q == p.q and ctx.P == p.P
    K, L, t = -(-M_ // p.slots), p.L, p.slots
    assert K == 123
    g = synth.rng(4242)
    ext = list(p.ext_mods())
    rlk = _uni_key(g, p, L, ext)
    ctx.import_switch_key(0, 0, _cuda(rlk))
    gk = {}
    for i in range(p.log_n - 1):
        key = _uni_key(g, p, L, ext)
        ctx.import_switch_key(1, 1 << i, _cuda(key))
        gk[oracle_mod.galois_elt(p, 1 << i)] = key
    Hc = _HCols(oracle_mod, p, K)
    Hd = ctx.alloc(N_COLS * K, 1, L, None, p.scale)
    for j in range(N_COLS):
        Hd.t[j * K:(j + 1) * K] = ctx.import_coeffs(_cuda(Hc.raw(j)[:, None]), L, p.scale).t
    O = np.stack([synth.uniform_residues(g, p.q[:L - 2], p.N) for _ in range(N_COLS)])
    Od = ctx.import_coeffs(_cuda(O[:, None]), L - 2, p.scale)
    model = ctx.privft_model_wrap(Hd, Od, M_, N_COLS, CLS)
    bag = ctx.alloc(BATCH * K, 2, L, None, p.scale)
    for b in range(BATCH):
        bag.t[b * K:(b + 1) * K] = ctx.import_coeffs(_cuda(_bag_raw(p, K, b)), L, p.scale).t
    w = [int(x) for x in g.integers(50, 601, size=BATCH)]
    scores = _host(ctx.export_coeffs(ctx.privft_infer(model, bag, w, True)))
    cd = ctx.privft_chunkdot(model, bag)
    pairs = [(b, j) for b in (0, 7, 19, 31) for j in range(0, N_COLS, 19)][:64]
    assert len(pairs) == 64
    got_cd = {bj: _host(ctx.export_coeffs(cd.view(bj[0] * N_COLS + bj[1], bj[0] * N_COLS + bj[1] + 1)))[0]
              for bj in pairs}
    del cd
    # oracle: the sampled chunk-dot outputs and one full query, on every host core
    _SAMPLE_CTX = (oracle_mod, p, K, Hc)
    with mp.get_context("fork").Pool(NPROC, initializer=oracle_mod.worker_init) as pool:
        want_cd = pool.map(_chunkdot_sample, pairs)
    for bj, (w0, w1) in zip(pairs, want_cd):
        assert np.array_equal(got_cd[bj][0], w0) and np.array_equal(got_cd[bj][1], w1), bj
    b0 = 7
    bag0 = _bag_raw(p, K, b0)
    cts = [oracle_mod.Ciphertext([bag0[k, 0], bag0[k, 1]], L, p.scale) for k in range(K)]
    O_pts = [oracle_mod.Plaintext(O[j], L - 2, p.scale) for j in range(N_COLS)]
    want = oracle_mod.privft_infer(p, cts, w[b0], Hc, O_pts, rlk, gk, True, workers=NPROC)
    assert np.array_equal(scores[b0, 0], want.c[0]) and np.array_equal(scores[b0, 1], want.c[1])
    ctx.close()
