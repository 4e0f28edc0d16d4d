"""oracle -- plain, slow CPU RNS-CKKS written from the paper.  TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product package
``paper_1908_06972_b200`` never imports it, and the two share no code: this module
and ``oracle/ckks_oracle.c`` re-derive every table, constant and step themselves.

Exact modular arithmetic lives in ``ckks_oracle.c`` (u64 residues, ``unsigned
__int128`` products reduced with ``%``); this file holds the floating-point
encode/decode (numpy FFT as a library primitive), the scheme-level orchestration
in the paper's order, and the float64 plaintext fastText reference.

Citations: ``P:NNN`` is /root/reference/PAPER.md line NNN; ``S:NNN`` is SPEC.md.
Ambiguity readings ``A1..A32`` are SURVEY.md Appendix A, restated in DESIGN.md.

Every function is pinned by a ``-m "not gpu"`` test (tests/test_oracle_*.py) against
something other than itself.  Functions without such a pin would say "parity
unpinned" here; there are none at present.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ckks_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

U64P = ctypes.POINTER(ctypes.c_uint64)
I64P = ctypes.POINTER(ctypes.c_int64)


def build(force: bool = False) -> str:
    """Compile the C oracle (gcc, -O2, OpenMP over independent limbs only)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-o", _LIB, _SRC])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        u32, u64 = ctypes.c_uint32, ctypes.c_uint64
        L.or_powmod.restype = u64
        L.or_powmod.argtypes = [u64, u64, u64]
        L.or_invmod.restype = u64
        L.or_invmod.argtypes = [u64, u64]
        L.or_is_prime.restype = ctypes.c_int
        L.or_is_prime.argtypes = [u64]
        L.or_prime_scan.restype = ctypes.c_int
        L.or_prime_scan.argtypes = [u32, u32, u32, u32, U64P]
        L.or_min_psi.restype = u64
        L.or_min_psi.argtypes = [u64, u32]
        for nm in ("or_ntt_fwd", "or_ntt_inv"):
            getattr(L, nm).restype = None
            getattr(L, nm).argtypes = [U64P, u32, u64, u64]
        for nm in ("or_poly_mul", "or_poly_add", "or_poly_sub"):
            getattr(L, nm).restype = None
            getattr(L, nm).argtypes = [U64P, U64P, U64P, U64P, u32, u32]
        L.or_poly_neg.restype = None
        L.or_poly_neg.argtypes = [U64P, U64P, U64P, u32, u32]
        L.or_poly_scalar_mul.restype = None
        L.or_poly_scalar_mul.argtypes = [U64P, U64P, U64P, U64P, u32, u32]
        L.or_poly_from_signed.restype = None
        L.or_poly_from_signed.argtypes = [I64P, U64P, U64P, u32, u32]
        L.or_automorphism.restype = None
        L.or_automorphism.argtypes = [U64P, U64P, U64P, u32, u32, u64]
        L.or_rescale_poly.restype = None
        L.or_rescale_poly.argtypes = [U64P, U64P, U64P, u32, u32]
        L.or_keyswitch.restype = None
        L.or_keyswitch.argtypes = [U64P, u32, U64P, u32, U64P, u32, U64P, U64P]
        U32P = ctypes.POINTER(ctypes.c_uint32)
        L.or_fast_bconv.restype = None
        L.or_fast_bconv.argtypes = [U64P, U32P, u32, U32P, u32, U64P, u32, U64P]
        L.or_keyswitch_hybrid.restype = None
        L.or_keyswitch_hybrid.argtypes = [U64P, u32, U64P, u32, u32, u32, U64P, u32, U64P, U64P]
        L.or_set_threads.restype = None
        L.or_set_threads.argtypes = [ctypes.c_int]
        _lib = L
    return _lib


def worker_init():
    """Initializer for forked worker processes: the parent's OpenMP pool does not survive
    fork(), so each worker runs the oracle's loops on one thread."""
    lib().or_set_threads(1)


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    if a.dtype == np.uint64:
        return a.ctypes.data_as(U64P)
    if a.dtype == np.int64:
        return a.ctypes.data_as(I64P)
    raise TypeError(a.dtype)


def _u64(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.uint64))


# ------------------------------------------------------------------ scalars --

def is_prime(n: int) -> bool:
    return bool(lib().or_is_prime(n))


def powmod(b: int, e: int, q: int) -> int:
    return int(lib().or_powmod(b, e, q))


def invmod(a: int, q: int) -> int:
    return int(lib().or_invmod(a, q))


def prime_scan(log_n: int, bits: int, skip: int, count: int) -> list[int]:
    out = np.zeros(max(count, 1), dtype=np.uint64)
    got = lib().or_prime_scan(log_n, bits, skip, count, _p(out))
    if got < count:
        raise ValueError(f"prime exhaustion: {got} < {count} primes = 1 mod 2N below 2^{bits}")
    return [int(x) for x in out[:count]]


def prime_chain(log_n: int, limb_bits: list[int], special_bits: int = 60, n_special: int = 1):
    """SURVEY O1 / Appendix C rule: one descending scan per bit size; the special
    prime(s) are drawn first from the special_bits scan, then each ciphertext prime
    in order from its own bits' scan.  Chain is decreasing ("ordered such
    that p_i < p_{i-1}")."""
    cursor: dict[int, int] = {}

    def take(bits):
        k = cursor.get(bits, 0)
        cursor[bits] = k + 1
        return prime_scan(log_n, bits, k, 1)[0]

    special = [take(special_bits) for _ in range(n_special)]
    qs = [take(b) for b in limb_bits]
    return qs, special


def min_psi(q: int, log_n: int) -> int:
    return int(lib().or_min_psi(q, log_n))


# ------------------------------------------------------------------- params --

@dataclass
class Params:
    """SETUP: ring degree N, prime chain q_0 > ... > q_{L-1}, special prime(s).
    Key switching (readings A6-A9): digits of `alpha` limbs, special primes `special`
    (default: the single prime P, alpha = 1).  alpha > 1 or several special primes is the
    hybrid key switching of SURVEY 8(f) row f2."""
    log_n: int
    q: list[int]                 # ciphertext primes q_0..q_{L-1}
    P0: int                      # first special prime (reading A6)
    scale: float                 # default Delta = 2^rho
    sigma: float = 3.2
    alpha: int = 1
    special: list | None = None

    def __post_init__(self):
        if self.special is None:
            self.special = [self.P0]

    @property
    def P(self) -> int:
        """P = product of the special primes."""
        return math.prod(self.special)

    @property
    def K(self) -> int:
        return len(self.special)

    @property
    def dnum(self) -> int:
        return -(-self.L // self.alpha)

    @property
    def N(self) -> int:
        return 1 << self.log_n

    @property
    def L(self) -> int:
        return len(self.q)

    @property
    def slots(self) -> int:
        return self.N // 2

    def mods(self, level: int) -> np.ndarray:
        return _u64(self.q[:level])

    def ext_mods(self) -> np.ndarray:
        """q_0..q_{L-1}, p_0..p_{K-1}: the key basis."""
        return _u64(self.q + list(self.special))


def preset(name: str) -> Params:
    """SURVEY Appendix C presets, re-derived by the oracle's own prime scan."""
    name = name.upper()
    if name == "C1":
        qs, sp = prime_chain(12, [30] * 3)
        return Params(12, qs, sp[0], 2.0 ** 30)
    if name == "C2":
        qs, sp = prime_chain(14, [40] * 8)
        return Params(14, qs, sp[0], 2.0 ** 40)
    if name == "C3":
        qs, sp = prime_chain(16, [40] * 30)
        return Params(16, qs, sp[0], 2.0 ** 40)
    if name == "C4":
        qs, sp = prime_chain(13, [60] + [40] * 4)
        return Params(13, qs, sp[0], 2.0 ** 40)
    raise KeyError(name)


def toy_params(log_n: int, limb_bits: list[int], special_bits: int = 60, scale: float = 2.0 ** 20,
               alpha: int = 1, n_special: int = 1) -> Params:
    qs, sp = prime_chain(log_n, limb_bits, special_bits, n_special)
    return Params(log_n, qs, sp[0], scale, alpha=alpha, special=sp)


# ------------------------------------------------------------- ring helpers --

def ntt_fwd(a, log_n: int, q: int, psi: int | None = None) -> np.ndarray:
    x = _u64(a).copy()
    lib().or_ntt_fwd(_p(x), log_n, q, psi if psi is not None else min_psi(q, log_n))
    return x


def ntt_inv(a, log_n: int, q: int, psi: int | None = None) -> np.ndarray:
    x = _u64(a).copy()
    lib().or_ntt_inv(_p(x), log_n, q, psi if psi is not None else min_psi(q, log_n))
    return x


def poly_mul(a, b, mods, log_n: int) -> np.ndarray:
    a, b, m = _u64(a), _u64(b), _u64(mods)
    out = np.empty_like(a)
    lib().or_poly_mul(_p(a), _p(b), _p(out), _p(m), len(m), log_n)
    return out


def poly_add(a, b, mods, log_n: int) -> np.ndarray:
    a, b, m = _u64(a), _u64(b), _u64(mods)
    out = np.empty_like(a)
    lib().or_poly_add(_p(a), _p(b), _p(out), _p(m), len(m), log_n)
    return out


def poly_sub(a, b, mods, log_n: int) -> np.ndarray:
    a, b, m = _u64(a), _u64(b), _u64(mods)
    out = np.empty_like(a)
    lib().or_poly_sub(_p(a), _p(b), _p(out), _p(m), len(m), log_n)
    return out


def poly_neg(a, mods, log_n: int) -> np.ndarray:
    a, m = _u64(a), _u64(mods)
    out = np.empty_like(a)
    lib().or_poly_neg(_p(a), _p(out), _p(m), len(m), log_n)
    return out


def poly_scalar_mul(a, c, mods, log_n: int) -> np.ndarray:
    a, c, m = _u64(a), _u64(c), _u64(mods)
    out = np.empty_like(a)
    lib().or_poly_scalar_mul(_p(a), _p(c), _p(out), _p(m), len(m), log_n)
    return out


def poly_from_signed(e, mods, log_n: int) -> np.ndarray:
    e = np.ascontiguousarray(np.asarray(e, dtype=np.int64))
    m = _u64(mods)
    out = np.empty((len(m), 1 << log_n), dtype=np.uint64)
    lib().or_poly_from_signed(_p(e), _p(out), _p(m), len(m), log_n)
    return out


def automorphism(a, kappa: int, mods, log_n: int) -> np.ndarray:
    a, m = _u64(a), _u64(mods)
    out = np.empty_like(a)
    lib().or_automorphism(_p(a), _p(out), _p(m), len(m), log_n, kappa)
    return out


def rescale_poly(c, mods, log_n: int) -> np.ndarray:
    c, m = _u64(c), _u64(mods)
    out = np.empty((len(m) - 1, 1 << log_n), dtype=np.uint64)
    lib().or_rescale_poly(_p(c), _p(out), _p(m), len(m), log_n)
    return out


def keyswitch(d, key, key_levels: int, ext_mods, log_n: int, alpha: int = 1, K: int = 1):
    """KS(d; key) -> (k0, k1), readings A6-A9 (see ckks_oracle.c); alpha > 1 or K > 1:
    hybrid key switching with fast base conversion."""
    d, key, m = _u64(d), _u64(key), _u64(ext_mods)
    level = d.shape[0]
    n = 1 << log_n
    o0 = np.empty((level, n), dtype=np.uint64)
    o1 = np.empty((level, n), dtype=np.uint64)
    if alpha == 1 and K == 1:
        lib().or_keyswitch(_p(d), level, _p(key), key_levels, _p(m), log_n, _p(o0), _p(o1))
    else:
        lib().or_keyswitch_hybrid(_p(d), level, _p(key), key_levels, K, alpha, _p(m), log_n, _p(o0), _p(o1))
    return o0, o1


def fast_bconv(x, src: list[int], tgt: list[int], mods, log_n: int) -> np.ndarray:
    """HPS fast base conversion of x (rows for the moduli indexed by src) to the moduli
    indexed by tgt: sum_i [x_i (Q/q_i)^{-1}]_{q_i} (Q/q_i) mod m_t (= x + u Q, 0 <= u < |src|)."""
    x, m = _u64(x), _u64(mods)
    s = np.ascontiguousarray(np.asarray(src, dtype=np.uint32))
    t = np.ascontiguousarray(np.asarray(tgt, dtype=np.uint32))
    out = np.empty((len(tgt), 1 << log_n), dtype=np.uint64)
    U32P = ctypes.POINTER(ctypes.c_uint32)
    lib().or_fast_bconv(_p(x), s.ctypes.data_as(U32P), len(src), t.ctypes.data_as(U32P), len(tgt), _p(m), log_n,
                        _p(out))
    return out


def crt_int(residues, mods) -> list[int]:
    """CRT recomposition to integers in [0, Q); Python big integers."""
    mods = [int(q) for q in mods]
    Q = math.prod(mods)
    res = np.asarray(residues)
    out = np.zeros(res.shape[1], dtype=object)
    for i, q in enumerate(mods):
        Qi = Q // q
        c = (Qi * pow(Qi % q, -1, q)) % Q
        out = out + res[i].astype(object) * c
    return [int(x) % Q for x in out]


def centered(xs, Q):
    return [x - Q if x > Q // 2 else x for x in xs]


# ------------------------------------------------------------ encode/decode --

def slot_exponents(log_n: int) -> np.ndarray:
    """r_j = 5^j mod 2N for j < N/2: slot j <-> root zeta^{r_j}, zeta = e^{i pi/N}
    (reading A12: rotation by pi = cyclic shift of the slots)."""
    n = 1 << log_n
    r = np.empty(n // 2, dtype=np.int64)
    x = 1
    for j in range(n // 2):
        r[j] = x
        x = (x * 5) % (2 * n)
    return r


def encode_coeffs(z, scale: float, log_n: int) -> np.ndarray:
    """ENCODE: mu = round(IDFT(Delta * z)) -- the inverse canonical embedding.
    Find real m(X) with m(zeta^{r_j}) = Delta z_j and m(zeta^{-r_j}) = conj(Delta z_j).
    With b_k = m_k zeta^k:  m(zeta^{2s+1}) = sum_k b_k omega^{s k}, omega = e^{2 pi i/N},
    so b = (1/N) * DFT^{-1} of the slot values (numpy fft as the library primitive).
    Coefficients are rounded half away from zero (reading A28)."""
    n = 1 << log_n
    z = _pad_slots(z, n // 2)
    r = slot_exponents(log_n)
    B = np.zeros(n, dtype=np.complex128)
    B[(r - 1) // 2] = scale * z
    B[(2 * n - r - 1) // 2] = np.conj(scale * z)
    b = np.fft.fft(B) / n
    k = np.arange(n)
    m = (b * np.exp(-1j * np.pi * k / n)).real
    return np.where(m >= 0, np.floor(m + 0.5), -np.floor(-m + 0.5)).astype(np.int64)


def _pad_slots(z, t):
    z = np.asarray(z, dtype=np.complex128).reshape(-1)
    if z.size > t:
        raise ValueError("overlong vector (S:170)")
    out = np.zeros(t, dtype=np.complex128)
    out[: z.size] = z
    return out


def decode_coeffs(m, scale: float, log_n: int) -> np.ndarray:
    """DECODE: v = DFT(mu / Delta): slot j = m(zeta^{r_j}) / Delta."""
    n = 1 << log_n
    m = np.asarray(m, dtype=np.float64)
    k = np.arange(n)
    b = m * np.exp(1j * np.pi * k / n)
    B = np.fft.ifft(b) * n
    r = slot_exponents(log_n)
    return B[(r - 1) // 2] / scale


# --------------------------------------------------------------- the scheme --

@dataclass
class Plaintext:
    m: np.ndarray          # [level][N] residues (coefficient form)
    level: int
    scale: float


@dataclass
class Ciphertext:
    c: list                # 2 (or 3) arrays [level][N], coefficient form
    level: int
    scale: float


@dataclass
class Keys:
    """KEYGEN outputs, coefficient form over q_0..q_{L-1}[, P]."""
    s: np.ndarray                         # int64 binary secret (reading A2)
    pk: tuple                             # (b, a), each [L][N]   (b = -a s + e)
    rlk: np.ndarray | None = None         # [L][2][L+1][N]
    gk: dict = field(default_factory=dict)  # kappa -> [L][2][L+1][N]


def encode(p: Params, z, level: int | None = None, scale: float | None = None) -> Plaintext:
    level = p.L if level is None else level
    scale = p.scale if scale is None else scale
    coeffs = encode_coeffs(z, scale, p.log_n)
    return Plaintext(poly_from_signed(coeffs, p.mods(level), p.log_n), level, scale)


def plain_to_ints(p: Params, pt_m: np.ndarray, level: int) -> list[int]:
    Q = math.prod(p.q[:level])
    return centered(crt_int(pt_m, p.q[:level]), Q)


def decode(p: Params, pt: Plaintext) -> np.ndarray:
    ints = plain_to_ints(p, pt.m, pt.level)
    return decode_coeffs(np.array([float(x) for x in ints]), pt.scale, p.log_n)


def keygen_public(p: Params, s, a, e) -> tuple:
    """pk = (b, a), b = -a s + e mod q_L.  a: [L][N] uniform residues,
    s: binary int poly, e: Gaussian int poly -- randomness supplied by the caller."""
    mods = p.mods(p.L)
    s_r = poly_from_signed(s, mods, p.log_n)
    e_r = poly_from_signed(e, mods, p.log_n)
    a = _u64(a)
    b = poly_add(poly_neg(poly_mul(a, s_r, mods, p.log_n), mods, p.log_n), e_r, mods, p.log_n)
    return (b, a)


def keygen_switch(p: Params, s, s_from_res: np.ndarray, a, e) -> np.ndarray:
    """Key-switching key s_from -> s (reading A6/A9; f2 for alpha > 1):
    for digit d < dnum = ceil(L/alpha), limb i in {q_0..q_{L-1}, p_0..p_{K-1}}:
        b_{d,i} = -a_{d,i} s + e_d + [i in digit d] (P mod q_i) s_from   (mod m_i)
    (P Q^_d s_from with Q^_d the CRT idempotent of the digit; alpha = 1: [i == d]).
    s_from_res: [L+K][N] residues of the source key (s^2 or phi_kappa(s)).
    a: [dnum][L+K][N] uniform residues; e: [dnum][N] Gaussian integers."""
    L, n, K = p.L, p.N, p.K
    em = p.ext_mods()
    s_r = poly_from_signed(s, em, p.log_n)
    key = np.empty((p.dnum, 2, L + K, n), dtype=np.uint64)
    a = _u64(a)
    for d in range(p.dnum):
        e_r = poly_from_signed(e[d], em, p.log_n)
        b = poly_add(poly_neg(poly_mul(a[d], s_r, em, p.log_n), em, p.log_n), e_r, em, p.log_n)
        for i in range(d * p.alpha, min(d * p.alpha + p.alpha, L)):
            q = p.q[i]
            term = (s_from_res[i].astype(object) * (p.P % q)) % q
            b[i] = poly_add(b[i:i + 1], _u64(term.astype(np.uint64))[None, :], [q], p.log_n)[0]
        key[d, 0] = b
        key[d, 1] = a[d]
    return key


def keygen_relin(p: Params, s, a, e) -> np.ndarray:
    """Relinearisation key s^2 -> s."""
    em = p.ext_mods()
    s_r = poly_from_signed(s, em, p.log_n)
    s2 = poly_mul(s_r, s_r, em, p.log_n)
    return keygen_switch(p, s, s2, a, e)


def galois_elt(p: Params, step: int) -> int:
    """kappa = 5^step mod 2N (left rotation for step > 0), 5^{-|step|} otherwise (A10)."""
    two_n = 2 * p.N
    k = pow(5, abs(step), two_n)
    return k if step >= 0 else pow(k, -1, two_n)


def keygen_galois(p: Params, s, step: int, a, e) -> tuple[int, np.ndarray]:
    """Rotation key phi_kappa(s) -> s (P:163 footnote)."""
    kappa = galois_elt(p, step)
    em = p.ext_mods()
    s_r = poly_from_signed(s, em, p.log_n)
    return kappa, keygen_switch(p, s, automorphism(s_r, kappa, em, p.log_n), a, e)


def encrypt(p: Params, pk, pt: Plaintext, u, e0, e1) -> Ciphertext:
    """ENC (garbled; reading A1): c0 = b u + mu + e0, c1 = a u + e1, u binary."""
    lv = pt.level
    mods = p.mods(lv)
    b, a = pk[0][:lv], pk[1][:lv]
    u_r = poly_from_signed(u, mods, p.log_n)
    c0 = poly_add(poly_add(poly_mul(b, u_r, mods, p.log_n), pt.m, mods, p.log_n),
                  poly_from_signed(e0, mods, p.log_n), mods, p.log_n)
    c1 = poly_add(poly_mul(a, u_r, mods, p.log_n), poly_from_signed(e1, mods, p.log_n), mods, p.log_n)
    return Ciphertext([c0, c1], lv, pt.scale)


def decrypt(p: Params, s, ct: Ciphertext) -> Plaintext:
    """DEC: mu = c0 + c1 s (+ c2 s^2 for a 3-part ciphertext, reading A29)."""
    mods = p.mods(ct.level)
    s_r = poly_from_signed(s, mods, p.log_n)
    acc = ct.c[0]
    spow = s_r
    for ci in ct.c[1:]:
        acc = poly_add(acc, poly_mul(ci, spow, mods, p.log_n), mods, p.log_n)
        spow = poly_mul(spow, s_r, mods, p.log_n)
    return Plaintext(acc, ct.level, ct.scale)


def _check_same(a: Ciphertext, b) -> None:
    if a.level != b.level:
        raise ValueError("level mismatch (A30)")


def add(p: Params, a: Ciphertext, b: Ciphertext) -> Ciphertext:
    """HADD; scales must be bitwise equal (A13)."""
    _check_same(a, b)
    if a.scale != b.scale:
        raise ValueError("scale mismatch (A13)")
    mods = p.mods(a.level)
    return Ciphertext([poly_add(x, y, mods, p.log_n) for x, y in zip(a.c, b.c)], a.level, a.scale)


def add_plain(p: Params, ct: Ciphertext, pt: Plaintext) -> Ciphertext:
    """HADDPLAIN: (c0 + pt, c1)."""
    _check_same(ct, pt)
    if ct.scale != pt.scale:
        raise ValueError("scale mismatch (A13)")
    mods = p.mods(ct.level)
    return Ciphertext([poly_add(ct.c[0], pt.m, mods, p.log_n)] + list(ct.c[1:]), ct.level, ct.scale)


def mul_plain(p: Params, ct: Ciphertext, pt: Plaintext) -> Ciphertext:
    """HMULPLAIN: (c0 pt, c1 pt); scale multiplies."""
    _check_same(ct, pt)
    mods = p.mods(ct.level)
    return Ciphertext([poly_mul(x, pt.m, mods, p.log_n) for x in ct.c], ct.level, ct.scale * pt.scale)


def const_residues(p: Params, value: float, const_scale: float, level: int) -> np.ndarray:
    """The constant polynomial llround(value * const_scale) (A15)."""
    c = _llround(value * const_scale)
    return _u64([c % q for q in p.q[:level]])


def _llround(x: float) -> int:
    return int(math.floor(x + 0.5)) if x >= 0 else -int(math.floor(-x + 0.5))


def mul_const(p: Params, ct: Ciphertext, value: float, const_scale: float) -> Ciphertext:
    c = const_residues(p, value, const_scale, ct.level)
    mods = p.mods(ct.level)
    return Ciphertext([poly_scalar_mul(x, c, mods, p.log_n) for x in ct.c], ct.level, ct.scale * const_scale)


def add_const(p: Params, ct: Ciphertext, value: float) -> Ciphertext:
    """Add the constant polynomial llround(value * ct.scale) to c0 (coefficient 0)."""
    c = const_residues(p, value, ct.scale, ct.level)
    c0 = ct.c[0].copy()
    for i, q in enumerate(p.q[:ct.level]):
        c0[i, 0] = (int(c0[i, 0]) + int(c[i])) % q
    return Ciphertext([c0] + list(ct.c[1:]), ct.level, ct.scale)


def tensor(p: Params, a: Ciphertext, b: Ciphertext) -> Ciphertext:
    """HMUL before relinearisation: (c00 c10, c00 c11 + c01 c10, c01 c11)."""
    _check_same(a, b)
    mods = p.mods(a.level)
    pm = lambda x, y: poly_mul(x, y, mods, p.log_n)
    d0 = pm(a.c[0], b.c[0])
    d1 = poly_add(pm(a.c[0], b.c[1]), pm(a.c[1], b.c[0]), mods, p.log_n)
    d2 = pm(a.c[1], b.c[1])
    return Ciphertext([d0, d1, d2], a.level, a.scale * b.scale)


def relinearize(p: Params, ct3: Ciphertext, rlk: np.ndarray) -> Ciphertext:
    """(d0, d1) + KS(d2; rlk) (reading A6)."""
    lv = ct3.level
    mods = p.mods(lv)
    k0, k1 = keyswitch(ct3.c[2], rlk, p.L, p.ext_mods(), p.log_n, p.alpha, p.K)
    return Ciphertext([poly_add(ct3.c[0], k0, mods, p.log_n), poly_add(ct3.c[1], k1, mods, p.log_n)],
                      lv, ct3.scale)


def mul_relin(p: Params, a: Ciphertext, b: Ciphertext, rlk: np.ndarray) -> Ciphertext:
    return relinearize(p, tensor(p, a, b), rlk)


def rescale(p: Params, ct: Ciphertext) -> Ciphertext:
    """RESCALE (Eq. 1, Alg "RNS RESCALE"); scale /= q_{l-1} (A13)."""
    if ct.level < 2:
        raise ValueError("level exhausted (S:206)")
    mods = p.mods(ct.level)
    return Ciphertext([rescale_poly(x, mods, p.log_n) for x in ct.c], ct.level - 1,
                      ct.scale / float(p.q[ct.level - 1]))


def naf(x: int) -> list[int]:
    """Non-adjacent form digits (LSB first) of x >= 0 (reading A10)."""
    out = []
    while x > 0:
        if x & 1:
            d = 2 - (x & 3)
            x -= d
        else:
            d = 0
        out.append(d)
        x >>= 1
    return out


def rotation_steps(p: Params, steps: int) -> list[int]:
    """Signed power-of-two rotations for `steps` (A10, A31): reduce mod t, NAF digits
    in increasing |2^i|; a digit of magnitude t is the identity and is dropped."""
    t = p.slots
    s = steps % t
    out = []
    for i, d in enumerate(naf(s)):
        if d and (1 << i) < t:
            out.append(d * (1 << i))
    return out


def apply_galois(p: Params, ct: Ciphertext, kappa: int, gkey: np.ndarray) -> Ciphertext:
    """One automorphism + key switch: (phi(c0) + k0, k1), (k0,k1) = KS(phi(c1); gk)."""
    mods = p.mods(ct.level)
    c0 = automorphism(ct.c[0], kappa, mods, p.log_n)
    c1 = automorphism(ct.c[1], kappa, mods, p.log_n)
    k0, k1 = keyswitch(c1, gkey, p.L, p.ext_mods(), p.log_n, p.alpha, p.K)
    return Ciphertext([poly_add(c0, k0, mods, p.log_n), k1], ct.level, ct.scale)


def rotate(p: Params, ct: Ciphertext, steps: int, gk: dict) -> Ciphertext:
    """ROTATE: left rotation by `steps` slots."""
    out = Ciphertext([x.copy() for x in ct.c], ct.level, ct.scale)
    for st in rotation_steps(p, steps):
        kappa = galois_elt(p, st)
        if kappa not in gk:
            raise KeyError(f"missing Galois key for step {st}")
        out = apply_galois(p, out, kappa, gk[kappa])
    return out


def total_sum(p: Params, ct: Ciphertext, gk: dict) -> Ciphertext:
    """Alg "TotalSum" with reading A11: for i = 0..log2(t)-1:
    ct <- ct + ROTATE(ct, 2^i)."""
    for i in range(p.log_n - 1):
        ct = add(p, ct, rotate(p, ct, 1 << i, gk))
    return ct


# -------------------------------------------------------------- PrivFT -------

def privft_column(p: Params, bag_chunks: list[Ciphertext], w: int, H_col: list[Plaintext], gk: dict) -> Ciphertext:
    """One embedding column j of the a8 sequence: h_j = rescale(TotalSum(rescale(
    sum_k HMULPLAIN(ct_k, P^H_{j,k}))) * llround(Delta/w))  (A14/A15)."""
    acc = None
    for k, ct in enumerate(bag_chunks):
        t = mul_plain(p, ct, H_col[k])
        acc = t if acc is None else add(p, acc, t)
    acc = rescale(p, acc)
    acc = total_sum(p, acc, gk)
    return rescale(p, mul_const(p, acc, 1.0 / w, p.scale))


_COL_ARGS = None


def _privft_column_worker(j: int) -> Ciphertext:
    p, bag_chunks, w, H_pts, gk = _COL_ARGS
    return privft_column(p, bag_chunks, w, H_pts[j], gk)


def privft_infer(p: Params, bag_chunks: list[Ciphertext], w: int, H_pts: list[list[Plaintext]],
                 O_pts: list[Plaintext], rlk, gk: dict, poly_softmax: bool, workers: int = 1) -> Ciphertext:
    """PrivFT encrypted inference, SURVEY 8(a) a8 sequence:
        a_j = sum_k HMULPLAIN(ct_k, P^H_{j,k});  rescale;  TotalSum;
        h_j = rescale(a_j * llround(Delta/w));  s = rescale(sum_j HMULPLAIN(h_j, P^O_j));
        [g = rescale(s*s + 4 s) + 2, scale *= 8  ==  s^2/8 + s/2 + 1/4]   (A19)
    workers > 1 maps the independent columns over forked processes (same arithmetic; used to
    keep the bench-shape parity test and the CPU baseline on every host core)."""
    cols = range(len(O_pts))
    if workers > 1:  # the n columns are independent ciphertexts (timing only: same arithmetic)
        import multiprocessing as mp
        global _COL_ARGS
        _COL_ARGS = (p, bag_chunks, w, H_pts, gk)
        with mp.get_context("fork").Pool(workers, initializer=worker_init) as pool:
            hs = pool.map(_privft_column_worker, cols)
        _COL_ARGS = None
    else:
        hs = [privft_column(p, bag_chunks, w, H_pts[j], gk) for j in cols]
    s = None
    for j, h in enumerate(hs):
        t = mul_plain(p, h, O_pts[j])
        s = t if s is None else add(p, s, t)
    s = rescale(p, s)
    if not poly_softmax:
        return s
    sq = mul_relin(p, s, s, rlk)
    lin = mul_const(p, s, 4.0, s.scale)
    g = rescale(p, add(p, sq, lin))
    g = add_const(p, g, 2.0)
    return Ciphertext(g.c, g.level, g.scale * 8.0)


def fasttext_plain(v: np.ndarray, w: int, H: np.ndarray, O: np.ndarray, poly_softmax: bool) -> np.ndarray:
    """float64 Alg "fasttext Inference" steps 2-3 plus the degree-2
    softmax polynomial X^2/8 + X/2 + 1/4."""
    h = (v.astype(np.float64) @ H) / w
    s = h @ O
    if poly_softmax:
        return s * s / 8 + s / 2 + 0.25
    return s


# ------------------------------------------------------- PrivFT training (f1) --
# Alg "GDMiniBatchTraining" with encrypted H and O ("the weight
# matrices here are encrypted, thus HMUL is used instead of HMULPLAIN"), the softmax
# polynomial and the error/gradient/update with mask and shift operations,
# realised as SPEC S:489/S:510 describe (readings T1-T6 in DESIGN.md):
#   per example (bag v: one chunk, m <= N/2; w tokens; label y, plaintext to the server):
#     a_j = rescale(HMULT(v, H_j)); a_j = TotalSum(a_j); h_j = rescale(a_j * 1/w)
#     s = rescale(relin(sum_j h_j (x) O_j)); g = rescale(s^2 + 4 s) + 2, scale *= 8
#     e = rescale(HMULPLAIN(g - onehot(y), mask_{<c}))
#     gO_j = rescale(HMULT(h_j, e));  gh_j = TotalSum(rescale(HMULT(O_j, e)))
#     gH_j = rescale(rescale(HMULT(v, gh_j)) * 1/w)
#   minibatch sums GH_j, GO_j (HADD), then H_j -= eta GH_j, O_j -= eta GO_j with eta a
#   constant whose scale is chosen so the product lands on the model's scale (T5); the
#   updated model is left at level l0 - 9: nine levels per minibatch.
def drop_level(ct: Ciphertext, level: int) -> Ciphertext:
    """Modulus drop (keep the first `level` limbs; message and scale unchanged)."""
    return Ciphertext([x[:level].copy() for x in ct.c], level, ct.scale)


def _const_to_scale(p: Params, ct: Ciphertext, value: float, target_scale: float) -> Ciphertext:
    """rescale(ct * value) with the constant's scale chosen so the result has scale
    target_scale; the tracked scale is then set to target_scale exactly (reading T5)."""
    cs = target_scale * float(p.q[ct.level - 1]) / ct.scale
    out = rescale(p, mul_const(p, ct, value, cs))
    return Ciphertext(out.c, out.level, target_scale)


def train_plaintexts(p: Params, H: list, O: list, examples: list, c: int):
    """-onehot(y) per example and the class mask, encoded at g's level and scale (the
    forward pass's scale bookkeeping, A13) so that they add to g exactly."""
    l0 = H[0].level
    sa = examples[0][0].scale * H[0].scale / float(p.q[l0 - 1])
    sh = sa * p.scale / float(p.q[l0 - 2])
    ss = sh * O[0].scale / float(p.q[l0 - 3])
    gs = ss * ss / float(p.q[l0 - 4]) * 8.0
    t = p.slots
    negs = []
    for (_, _, y) in examples:
        z = np.zeros(t)
        z[y] = -1.0
        negs.append(encode(p, z, level=l0 - 4, scale=gs))
    z = np.zeros(t)
    z[:c] = 1.0
    return negs, encode(p, z, level=l0 - 4, scale=p.scale)


def train_gradients(p: Params, H: list, O: list, examples: list, c: int, rlk, gk: dict, plaintexts=None):
    """Encrypted gradient sums over one minibatch: returns (GH [n], GO [n]).
    plaintexts: (neg_onehots, mask) from train_plaintexts (encoded here if None)."""
    negs, mask_pt = plaintexts if plaintexts is not None else train_plaintexts(p, H, O, examples, c)
    l0 = H[0].level
    GH = GO = None
    for ex_i, (v, w, y) in enumerate(examples):
        a = [total_sum(p, rescale(p, mul_relin(p, v, Hj, rlk)), gk) for Hj in H]
        h = [rescale(p, mul_const(p, aj, 1.0 / w, p.scale)) for aj in a]
        s3 = None  # sum_j h_j O_j accumulated as 3-part ciphertexts, relinearised once (T3)
        for hj, Oj in zip(h, O):
            x = tensor(p, hj, drop_level(Oj, l0 - 2))
            s3 = x if s3 is None else Ciphertext([poly_add(u, w_, p.mods(x.level), p.log_n)
                                                  for u, w_ in zip(s3.c, x.c)], x.level, x.scale)
        s = rescale(p, relinearize(p, s3, rlk))
        g = rescale(p, add(p, mul_relin(p, s, s, rlk), mul_const(p, s, 4.0, s.scale)))
        g = add_const(p, g, 2.0)
        g = Ciphertext(g.c, g.level, g.scale * 8.0)
        assert negs[ex_i].scale == g.scale and negs[ex_i].level == g.level
        e = rescale(p, mul_plain(p, add_plain(p, g, negs[ex_i]), mask_pt))
        gO = [rescale(p, mul_relin(p, drop_level(hj, e.level), e, rlk)) for hj in h]
        gh = [total_sum(p, rescale(p, mul_relin(p, drop_level(Oj, e.level), e, rlk)), gk) for Oj in O]
        vv = drop_level(v, gh[0].level)
        gH = [rescale(p, mul_const(p, rescale(p, mul_relin(p, vv, ghj, rlk)), 1.0 / w, p.scale)) for ghj in gh]
        GH = gH if GH is None else [add(p, x, y_) for x, y_ in zip(GH, gH)]
        GO = gO if GO is None else [add(p, x, y_) for x, y_ in zip(GO, gO)]
    return GH, GO


def train_update(p: Params, H: list, O: list, GH: list, GO: list, eta: float):
    """H_j -= eta GH_j, O_j -= eta GO_j; both left at level l0 - 9 (T4)."""
    l0 = H[0].level
    lf = l0 - 9
    Hn, On = [], []
    for Hj, gj in zip(H, GH):
        d = _const_to_scale(p, gj, -eta, Hj.scale)
        Hn.append(add(p, drop_level(Hj, d.level), d))
    for Oj, gj in zip(O, GO):
        d = _const_to_scale(p, gj, -eta, Oj.scale)
        On.append(drop_level(add(p, drop_level(Oj, d.level), d), lf))
    assert all(x.level == lf for x in Hn + On)
    return Hn, On


def train_plain(H: np.ndarray, O: np.ndarray, examples: list, c: int, eta: float):
    """float64 minibatch GD step (Alg "GDMiniBatchTraining" body) with the
    polynomial in place of softmax and e = g - onehot (masked to the c classes)."""
    GH = np.zeros_like(H)
    GO = np.zeros_like(O)
    for (v, w, y) in examples:
        h = v @ H / w
        s = h @ O
        g = s * s / 8 + s / 2 + 0.25
        e = g.copy()
        e[y] -= 1.0
        GO += np.outer(h, e)
        gh = O @ e
        GH += np.outer(v, gh) / w
    return H - eta * GH, O - eta * GO
