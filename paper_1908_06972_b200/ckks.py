"""Thin ctypes binding of libckks (include/ckks.h) -- argument marshalling only.

Every function named ``ckks_*`` here forwards to the C ABI function of the same name;
every arithmetic step runs in the sm_100a kernels of ``libckks.so``.  torch supplies
device memory (``Buf.t`` is a CUDA uint64 tensor) and the stream handle.  There is no
CPU fallback: importing this module without the built library raises.

``Context`` is a convenience wrapper that allocates output buffers and checks status.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# CKKS_LIB_VARIANT=<tag> loads libckks_<tag>.so (an A/B build from build.build(variant=...))
LIB_PATH = os.path.join(_HERE, f"libckks_{os.environ['CKKS_LIB_VARIANT']}.so" if os.environ.get("CKKS_LIB_VARIANT")
                        else "libckks.so")

c_u32, c_u64, c_i32, c_dbl, c_vp = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int32, ctypes.c_double, ctypes.c_void_p

STATUS = {0: "CKKS_OK", -1: "CKKS_E_INVALID_ARG", -2: "CKKS_E_LEVEL_MISMATCH", -3: "CKKS_E_SCALE_MISMATCH",
          -4: "CKKS_E_LEVEL_EXHAUSTED", -5: "CKKS_E_MISSING_KEY", -6: "CKKS_E_PRIME_EXHAUSTED",
          -7: "CKKS_E_ENCODE_OVERFLOW", -8: "CKKS_E_CUDA", -9: "CKKS_E_OOM", -10: "CKKS_E_UNSUPPORTED"}
POLY_SOFTMAX = 1


class CkksBuf(ctypes.Structure):
    _fields_ = [("data", c_vp), ("count", c_u32), ("n_polys", c_u32), ("level", c_u32), ("capacity", c_u32),
                ("scale", c_dbl)]


class CkksParams(ctypes.Structure):
    _fields_ = [("log_n", c_u32), ("n_limbs", c_u32), ("limb_bits", ctypes.POINTER(c_u32)), ("special_bits", c_u32),
                ("primes", ctypes.POINTER(c_u64)), ("scale", c_dbl), ("n_special", c_u32), ("digit_limbs", c_u32)]


P = ctypes.POINTER
BUFP = P(CkksBuf)
# name -> (restype, argtypes) ; mirrors include/ckks.h
_SIGS = {
    "ckks_ctx_create": (ctypes.c_int, [P(CkksParams), ctypes.c_int, c_vp, P(c_vp)]),
    "ckks_ctx_destroy": (ctypes.c_int, [c_vp]),
    "ckks_set_stream": (ctypes.c_int, [c_vp, c_vp]),
    "ckks_ctx_info": (ctypes.c_int, [c_vp, P(c_u32), P(c_u32), P(c_u64)]),
    "ckks_last_error": (ctypes.c_char_p, [c_vp]),
    "ckks_launch_count": (c_u64, [c_vp]),
    "ckks_profile_enable": (ctypes.c_int, [c_vp, ctypes.c_int]),
    "ckks_profile_read": (ctypes.c_int, [c_vp, P(ctypes.c_char_p), P(c_dbl), P(c_u64), P(c_dbl), c_u32, P(c_u32),
                                         ctypes.c_int]),
    "ckks_set_secret": (ctypes.c_int, [c_vp, c_vp]),
    "ckks_keygen_public": (ctypes.c_int, [c_vp, c_vp, c_vp]),
    "ckks_keygen_relin": (ctypes.c_int, [c_vp, c_vp, c_vp]),
    "ckks_keygen_galois": (ctypes.c_int, [c_vp, c_i32, c_vp, c_vp]),
    "ckks_import_switch_key": (ctypes.c_int, [c_vp, ctypes.c_int, c_i32, c_vp]),
    "ckks_galois_elt": (c_u64, [c_vp, c_i32]),
    "ckks_import_coeffs": (ctypes.c_int, [c_vp, c_vp, BUFP]),
    "ckks_export_coeffs": (ctypes.c_int, [c_vp, BUFP, c_vp]),
    "ckks_ntt": (ctypes.c_int, [c_vp, c_vp, c_u32, c_u32, ctypes.c_int]),
    "ckks_export": (ctypes.c_int, [c_vp, BUFP, c_vp, ctypes.c_size_t, P(ctypes.c_size_t)]),
    "ckks_import_info": (ctypes.c_int, [c_vp, c_vp, ctypes.c_size_t, P(c_u32), P(c_u32), P(c_u32), P(c_dbl)]),
    "ckks_import": (ctypes.c_int, [c_vp, c_vp, ctypes.c_size_t, BUFP]),
    "ckks_export_keys": (ctypes.c_int, [c_vp, c_vp, ctypes.c_size_t, P(ctypes.c_size_t)]),
    "ckks_import_keys": (ctypes.c_int, [c_vp, c_vp, ctypes.c_size_t]),
    "ckks_encode": (ctypes.c_int, [c_vp, P(c_dbl), P(c_dbl), ctypes.c_size_t, c_dbl, c_u32, BUFP]),
    "ckks_decode": (ctypes.c_int, [c_vp, BUFP, P(c_dbl), P(c_dbl), ctypes.c_size_t]),
    "ckks_encode_batch": (ctypes.c_int, [c_vp, c_vp, ctypes.c_size_t, c_dbl, c_u32, BUFP]),
    "ckks_ipc_export": (ctypes.c_int, [c_vp, c_vp, c_vp, P(c_u64)]),
    "ckks_ipc_open": (ctypes.c_int, [c_vp, c_vp, c_u64, P(c_vp)]),
    "ckks_ipc_close": (ctypes.c_int, [c_vp, c_vp]),
    "ckks_p2p_modsum": (ctypes.c_int, [c_vp, P(c_vp), P(c_vp), c_u32, c_u32, BUFP]),
    "ckks_decode_batch": (ctypes.c_int, [c_vp, BUFP, c_vp, ctypes.c_size_t]),
    "ckks_encode_overflowed": (ctypes.c_int, [c_vp, P(ctypes.c_int)]),
    "ckks_encrypt": (ctypes.c_int, [c_vp, BUFP, c_vp, c_vp, c_vp, BUFP]),
    "ckks_decrypt": (ctypes.c_int, [c_vp, BUFP, BUFP]),
    "ckks_add": (ctypes.c_int, [c_vp, BUFP, BUFP, BUFP]),
    "ckks_sub": (ctypes.c_int, [c_vp, BUFP, BUFP, BUFP]),
    "ckks_add_plain": (ctypes.c_int, [c_vp, BUFP, BUFP, BUFP]),
    "ckks_mul_plain": (ctypes.c_int, [c_vp, BUFP, BUFP, BUFP]),
    "ckks_mul_const": (ctypes.c_int, [c_vp, BUFP, c_dbl, c_dbl, BUFP]),
    "ckks_add_const": (ctypes.c_int, [c_vp, BUFP, c_dbl, BUFP]),
    "ckks_mul_relin": (ctypes.c_int, [c_vp, BUFP, BUFP, BUFP]),
    "ckks_rescale": (ctypes.c_int, [c_vp, BUFP, BUFP]),
    "ckks_mul_relin_rescale": (ctypes.c_int, [c_vp, BUFP, BUFP, BUFP]),
    "ckks_rotate": (ctypes.c_int, [c_vp, BUFP, c_i32, BUFP]),
    "ckks_total_sum": (ctypes.c_int, [c_vp, BUFP, BUFP]),
    "ckks_modadd_gathered": (ctypes.c_int, [c_vp, c_vp, c_u32, BUFP]),
    "ckks_shard_ks_digits": (ctypes.c_int, [c_vp, ctypes.c_int, c_i32, BUFP, BUFP, c_u32, c_u32, c_u32, BUFP, c_vp]),
    "ckks_shard_ks_finish": (ctypes.c_int, [c_vp, ctypes.c_int, c_i32, c_vp, c_u32, c_u32, BUFP, c_u32, c_u32, BUFP]),
    "ckks_shard_ks_window": (ctypes.c_int, [c_vp, ctypes.c_int, c_i32, c_vp, c_u32, c_u32, BUFP, c_u32, c_u32,
                                            ctypes.c_int]),
    "ckks_shard_ks_combine": (ctypes.c_int, [c_vp, ctypes.c_int, c_i32, BUFP, c_u32, c_u32, BUFP]),
    "ckks_shard_rescale_last": (ctypes.c_int, [c_vp, BUFP, c_u32, c_u32, c_vp]),
    "ckks_shard_rescale_apply": (ctypes.c_int, [c_vp, c_vp, BUFP, c_u32, c_u32, BUFP]),
    "ckks_privft_train_plan": (ctypes.c_int, [c_vp, BUFP, BUFP, BUFP, P(c_dbl), P(c_u32)]),
    "ckks_privft_train_grad": (ctypes.c_int, [c_vp, BUFP, BUFP, BUFP, P(c_u32), P(c_u32), c_u32, BUFP, BUFP, BUFP,
                                              BUFP]),
    "ckks_privft_train_update": (ctypes.c_int, [c_vp, BUFP, BUFP, BUFP, BUFP, c_dbl, BUFP, BUFP]),
    "ckks_privft_model_create": (ctypes.c_int, [c_vp, P(c_dbl), P(c_dbl), c_u32, c_u32, c_u32, P(c_vp)]),
    "ckks_privft_model_wrap": (ctypes.c_int, [c_vp, BUFP, BUFP, c_u32, c_u32, c_u32, P(c_vp)]),
    "ckks_privft_model_destroy": (ctypes.c_int, [c_vp]),
    "ckks_privft_chunkdot": (ctypes.c_int, [c_vp, c_vp, BUFP, c_u32, BUFP]),
    "ckks_privft_infer": (ctypes.c_int, [c_vp, c_vp, BUFP, P(c_u32), c_u32, c_u32, BUFP]),
    "ckks_privft_infer_host": (ctypes.c_int, [c_vp, c_vp, c_vp, c_dbl, P(c_u32), c_u32, c_u32, c_vp, P(c_dbl),
                                              P(c_u32)]),
    "ckks_sync": (ctypes.c_int, [c_vp]),
}
EXPORTS = tuple(_SIGS)

_lib = None


def lib() -> ctypes.CDLL:
    """Load libckks.so (fails loudly if it was not built -- there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                               "(python -m paper_1908_06972_b200.build); there is no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype, f.argtypes = res, args
        _lib = L
    return _lib


class CkksError(RuntimeError):
    pass


def _ptr(t: torch.Tensor | None):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


@dataclass
class Buf:
    """A batch of plaintexts / ciphertexts in caller-owned device memory (torch)."""
    t: torch.Tensor          # int64 view of uint64 words, shape [count, n_polys, capacity, N]
    level: int
    scale: float

    @property
    def count(self):
        return self.t.shape[0]

    @property
    def n_polys(self):
        return self.t.shape[1]

    @property
    def capacity(self):
        return self.t.shape[2]

    def c(self) -> CkksBuf:
        assert self.t.is_cuda and self.t.is_contiguous()
        return CkksBuf(self.t.data_ptr(), self.count, self.n_polys, self.level, self.capacity, self.scale)

    def sync(self, cb: CkksBuf) -> "Buf":
        self.level, self.scale = cb.level, cb.scale
        return self

    def view(self, start: int, stop: int) -> "Buf":
        return Buf(self.t[start:stop], self.level, self.scale)


class Context:
    """Owns a ckks_ctx on one CUDA device; all calls are stream-ordered on torch's current stream."""

    def __init__(self, log_n: int, limb_bits: list[int] | None = None, special_bits: int = 60,
                 scale: float = 2.0 ** 40, primes: list[int] | None = None, device: int = 0,
                 n_special: int = 1, digit_limbs: int = 1):
        """primes (optional): explicit q_0..q_{L-1} followed by the n_special special primes."""
        self.L_ = lib()
        torch.cuda.set_device(device)
        self.device = torch.device("cuda", device)
        nl = len(primes) - n_special if primes is not None else len(limb_bits)
        bits = (c_u32 * max(nl, 1))(*(limb_bits or [0] * nl))
        pr = (c_u64 * (nl + n_special))(*primes) if primes is not None else None
        prm = CkksParams(log_n, nl, ctypes.cast(bits, P(c_u32)), special_bits,
                         ctypes.cast(pr, P(c_u64)) if pr is not None else None, scale, n_special, digit_limbs)
        h = c_vp()
        st = torch.cuda.current_stream(self.device).cuda_stream
        rc = self.L_.ckks_ctx_create(ctypes.byref(prm), device, c_vp(st), ctypes.byref(h))
        if rc != 0:
            raise CkksError(f"ckks_ctx_create: {STATUS.get(rc, rc)}")
        self.h = h
        self._keep, self._host_calls = [None, None], 0
        self.log_n, self.N, self.L, self.scale = log_n, 1 << log_n, nl, scale
        self.K, self.alpha = n_special, digit_limbs
        self.dnum = -(-nl // digit_limbs)
        out = (c_u64 * (nl + n_special))()
        self.L_.ckks_ctx_info(self.h, None, None, out)
        self.primes = [int(x) for x in out]
        self.q, self.special = self.primes[:nl], self.primes[nl:]
        self.P = self.special[0] if n_special == 1 else self.special  # single special prime: the int

    def close(self):
        if getattr(self, "h", None):
            self.L_.ckks_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- plumbing -------------------------------------------------------------------
    def _chk(self, rc: int, what: str):
        if rc != 0:
            msg = self.L_.ckks_last_error(self.h).decode()
            raise CkksError(f"{what}: {STATUS.get(rc, rc)} {msg}")

    def set_stream(self, stream: torch.cuda.Stream | None = None):
        s = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        self._chk(self.L_.ckks_set_stream(self.h, c_vp(s)), "ckks_set_stream")

    def launches(self) -> int:
        return int(self.L_.ckks_launch_count(self.h))

    def profile(self, on: bool = True):
        self._chk(self.L_.ckks_profile_enable(self.h, int(on)), "ckks_profile_enable")

    def profile_read(self, reset: bool = True) -> dict:
        """{kernel: dict(ms, launches, bfly, mac, bytes, fbfly, fmac)} accumulated while profiling was on."""
        n = c_u32()
        self._chk(self.L_.ckks_profile_read(self.h, None, None, None, None, 0, ctypes.byref(n), 0),
                  "ckks_profile_read")
        k = n.value
        names = (ctypes.c_char_p * max(k, 1))()
        ms = (c_dbl * max(k, 1))()
        cnt = (c_u64 * max(k, 1))()
        work = (c_dbl * (5 * max(k, 1)))()
        self._chk(self.L_.ckks_profile_read(self.h, names, ms, cnt, work, k, ctypes.byref(n), int(reset)),
                  "ckks_profile_read")
        return {names[i].decode(): dict(ms=ms[i], launches=int(cnt[i]), bfly=work[5 * i], mac=work[5 * i + 1],
                                        bytes=work[5 * i + 2], fbfly=work[5 * i + 3], fmac=work[5 * i + 4])
                for i in range(k)}

    def alloc(self, count: int, n_polys: int, level: int, capacity: int | None = None, scale: float = 1.0) -> Buf:
        cap = capacity or level
        t = torch.empty((count, n_polys, cap, self.N), dtype=torch.int64, device=self.device)
        return Buf(t, level, scale)

    def galois_elt(self, step: int) -> int:
        return int(self.L_.ckks_galois_elt(self.h, step))

    # ---- keys ---------------------------------------------------------------------------
    def set_secret(self, s: torch.Tensor):
        self._chk(self.L_.ckks_set_secret(self.h, _ptr(s)), "ckks_set_secret")

    def keygen_public(self, a: torch.Tensor, e: torch.Tensor):
        self._chk(self.L_.ckks_keygen_public(self.h, _ptr(a), _ptr(e)), "ckks_keygen_public")

    def keygen_relin(self, a: torch.Tensor, e: torch.Tensor):
        self._chk(self.L_.ckks_keygen_relin(self.h, _ptr(a), _ptr(e)), "ckks_keygen_relin")

    def keygen_galois(self, step: int, a: torch.Tensor, e: torch.Tensor):
        self._chk(self.L_.ckks_keygen_galois(self.h, step, _ptr(a), _ptr(e)), "ckks_keygen_galois")

    def import_switch_key(self, kind: int, step: int, key_coeff: torch.Tensor):
        self._chk(self.L_.ckks_import_switch_key(self.h, kind, step, _ptr(key_coeff)), "ckks_import_switch_key")

    # ---- boundary -------------------------------------------------------------------------
    def import_coeffs(self, coeffs: torch.Tensor, level: int, scale: float, capacity: int | None = None) -> Buf:
        """coeffs: CUDA int64 [count, n_polys, level, N] coefficient-form canonical residues."""
        coeffs = coeffs.contiguous()
        b = self.alloc(coeffs.shape[0], coeffs.shape[1], level, capacity, scale)
        cb = b.c()
        self._chk(self.L_.ckks_import_coeffs(self.h, _ptr(coeffs), ctypes.byref(cb)), "ckks_import_coeffs")
        return b

    def export_coeffs(self, b: Buf) -> torch.Tensor:
        out = torch.empty((b.count, b.n_polys, b.level, self.N), dtype=torch.int64, device=self.device)
        cb = b.c()
        self._chk(self.L_.ckks_export_coeffs(self.h, ctypes.byref(cb), _ptr(out)), "ckks_export_coeffs")
        return out

    def export(self, b: Buf) -> bytes:
        """ckks_export: the serialised host bytes of b (coefficient form + header)."""
        n = ctypes.c_size_t()
        cb = b.c()
        self._chk(self.L_.ckks_export(self.h, ctypes.byref(cb), None, 0, ctypes.byref(n)), "ckks_export")
        out = ctypes.create_string_buffer(n.value)
        self._chk(self.L_.ckks_export(self.h, ctypes.byref(cb), out, n.value, ctypes.byref(n)), "ckks_export")
        return out.raw[:n.value]

    def import_bytes(self, data: bytes, capacity: int | None = None) -> Buf:
        """ckks_import_info + ckks_import: a new Buf holding the serialised ciphertexts/plaintexts."""
        cnt, npl, lev, sc = c_u32(), c_u32(), c_u32(), c_dbl()
        self._chk(self.L_.ckks_import_info(self.h, data, len(data), ctypes.byref(cnt), ctypes.byref(npl),
                                           ctypes.byref(lev), ctypes.byref(sc)), "ckks_import_info")
        b = self.alloc(cnt.value, npl.value, lev.value, capacity, sc.value)
        cb = b.c()
        self._chk(self.L_.ckks_import(self.h, data, len(data), ctypes.byref(cb)), "ckks_import")
        return b.sync(cb)

    def export_keys(self) -> bytes:
        n = ctypes.c_size_t()
        self._chk(self.L_.ckks_export_keys(self.h, None, 0, ctypes.byref(n)), "ckks_export_keys")
        out = ctypes.create_string_buffer(n.value)
        self._chk(self.L_.ckks_export_keys(self.h, out, n.value, ctypes.byref(n)), "ckks_export_keys")
        return out.raw[:n.value]

    def import_keys(self, data: bytes):
        self._chk(self.L_.ckks_import_keys(self.h, data, len(data)), "ckks_import_keys")

    def ntt(self, data: torch.Tensor, inverse: bool = False):
        """In-place batched NTT of data [count, level, N] (limb i mod q_i)."""
        assert data.is_contiguous()
        self._chk(self.L_.ckks_ntt(self.h, _ptr(data), data.shape[0], data.shape[1], int(inverse)), "ckks_ntt")

    # ---- encode/decode ------------------------------------------------------------------
    def encode(self, z, level: int | None = None, scale: float | None = None, capacity: int | None = None) -> Buf:
        level = self.L if level is None else level
        scale = self.scale if scale is None else scale
        z = np.asarray(z)
        re = np.ascontiguousarray(z.real, dtype=np.float64)
        im = np.ascontiguousarray(z.imag, dtype=np.float64) if np.iscomplexobj(z) else None
        b = self.alloc(1, 1, level, capacity, scale)
        cb = b.c()
        self._chk(self.L_.ckks_encode(self.h, re.ctypes.data_as(P(c_dbl)),
                                      im.ctypes.data_as(P(c_dbl)) if im is not None else None, re.size, scale,
                                      level, ctypes.byref(cb)), "ckks_encode")
        return b.sync(cb)

    def decode(self, pt: Buf, n_slots: int | None = None) -> np.ndarray:
        n_slots = self.N // 2 if n_slots is None else n_slots
        re = np.zeros(n_slots)
        im = np.zeros(n_slots)
        cb = pt.c()
        self._chk(self.L_.ckks_decode(self.h, ctypes.byref(cb), re.ctypes.data_as(P(c_dbl)),
                                      im.ctypes.data_as(P(c_dbl)), n_slots), "ckks_decode")
        return re + 1j * im

    def encode_batch(self, z: torch.Tensor, level: int | None = None, scale: float | None = None,
                     capacity: int | None = None, out: Buf | None = None) -> Buf:
        """GPU encode (f4): z CUDA complex128 (or float64) [count, n_slots] -> count plaintexts."""
        level = self.L if level is None else level
        scale = self.scale if scale is None else scale
        if not z.is_complex():
            z = z.to(torch.float64).to(torch.complex128)
        assert z.dtype == torch.complex128 and z.dim() == 2 and z.is_cuda
        z = z.contiguous()
        b = out if out is not None else self.alloc(z.shape[0], 1, level, capacity, scale)
        cb = b.c()
        self._chk(self.L_.ckks_encode_batch(self.h, _ptr(torch.view_as_real(z)), z.shape[1], scale, level,
                                            ctypes.byref(cb)), "ckks_encode_batch")
        return b.sync(cb)

    def decode_batch(self, pt: Buf, n_slots: int | None = None, out: torch.Tensor | None = None) -> torch.Tensor:
        """GPU decode (f4): count plaintexts -> CUDA complex128 [count, n_slots]."""
        n_slots = self.N // 2 if n_slots is None else n_slots
        z = out if out is not None else torch.empty((pt.count, n_slots), dtype=torch.complex128, device=self.device)
        cb = pt.c()
        self._chk(self.L_.ckks_decode_batch(self.h, ctypes.byref(cb), _ptr(torch.view_as_real(z)), n_slots),
                  "ckks_decode_batch")
        return z

    # ---- fused peer-memory modular all-reduce (f3) ---------------------------------------
    IPC_HANDLE_BYTES = 64

    def ipc_export(self, t: torch.Tensor) -> tuple[bytes, int]:
        h = ctypes.create_string_buffer(self.IPC_HANDLE_BYTES)
        off = c_u64(0)
        self._chk(self.L_.ckks_ipc_export(self.h, c_vp(t.data_ptr()), h, ctypes.byref(off)), "ckks_ipc_export")
        return h.raw, int(off.value)

    def ipc_open(self, handle: bytes, offset: int) -> int:
        p = c_vp(0)
        self._chk(self.L_.ckks_ipc_open(self.h, ctypes.create_string_buffer(handle, len(handle)), offset,
                                        ctypes.byref(p)), "ckks_ipc_open")
        return int(p.value)

    def ipc_close(self, ptr: int):
        self._chk(self.L_.ckks_ipc_close(self.h, c_vp(ptr)), "ckks_ipc_close")

    def p2p_modsum(self, in_ptrs: list[int], out_ptrs: list[int], rank: int, shape: Buf):
        R = len(in_ptrs)
        ins, outs = (c_vp * R)(*in_ptrs), (c_vp * R)(*out_ptrs)
        cb = shape.c()
        self._chk(self.L_.ckks_p2p_modsum(self.h, ins, outs, R, rank, ctypes.byref(cb)), "ckks_p2p_modsum")

    def encode_overflowed(self) -> bool:
        f = ctypes.c_int(0)
        self._chk(self.L_.ckks_encode_overflowed(self.h, ctypes.byref(f)), "ckks_encode_overflowed")
        return bool(f.value)

    def encrypt(self, pt: Buf, u: torch.Tensor, e0: torch.Tensor, e1: torch.Tensor,
                capacity: int | None = None) -> Buf:
        ct = self.alloc(pt.count, 2, pt.level, capacity, pt.scale)
        cb, pb = ct.c(), pt.c()
        self._chk(self.L_.ckks_encrypt(self.h, ctypes.byref(pb), _ptr(u), _ptr(e0), _ptr(e1), ctypes.byref(cb)),
                  "ckks_encrypt")
        return ct.sync(cb)

    def decrypt(self, ct: Buf) -> Buf:
        pt = self.alloc(ct.count, 1, ct.level, None, ct.scale)
        cb, pb = ct.c(), pt.c()
        self._chk(self.L_.ckks_decrypt(self.h, ctypes.byref(cb), ctypes.byref(pb)), "ckks_decrypt")
        return pt.sync(pb)

    # ---- ops ------------------------------------------------------------------------------
    def _out(self, like: Buf, out: Buf | None, level=None):
        return out if out is not None else self.alloc(like.count, 2, level or like.level, None, like.scale)

    def _op2(self, name, a: Buf, b: Buf, out: Buf | None):
        out = self._out(a, out)
        ca, cb, co = a.c(), b.c(), out.c()
        self._chk(getattr(self.L_, name)(self.h, ctypes.byref(ca), ctypes.byref(cb), ctypes.byref(co)), name)
        return out.sync(co)

    def add(self, a, b, out=None):
        return self._op2("ckks_add", a, b, out)

    def sub(self, a, b, out=None):
        return self._op2("ckks_sub", a, b, out)

    def add_plain(self, ct, pt, out=None):
        return self._op2("ckks_add_plain", ct, pt, out)

    def mul_plain(self, ct, pt, out=None):
        return self._op2("ckks_mul_plain", ct, pt, out)

    def mul_relin(self, a, b, out=None):
        return self._op2("ckks_mul_relin", a, b, out)

    def mul_const(self, ct: Buf, value: float, const_scale: float, out=None):
        out = self._out(ct, out)
        ca, co = ct.c(), out.c()
        self._chk(self.L_.ckks_mul_const(self.h, ctypes.byref(ca), value, const_scale, ctypes.byref(co)),
                  "ckks_mul_const")
        return out.sync(co)

    def add_const(self, ct: Buf, value: float, out=None):
        out = self._out(ct, out)
        ca, co = ct.c(), out.c()
        self._chk(self.L_.ckks_add_const(self.h, ctypes.byref(ca), value, ctypes.byref(co)), "ckks_add_const")
        return out.sync(co)

    def mul_relin_rescale(self, a, b, out=None):
        """HMult + relinearisation + rescale in one call (fused ModDown + rescale, reading A7)."""
        out = out if out is not None else self.alloc(a.count, 2, a.level - 1, a.level, 1.0)
        ca, cb, co = a.c(), b.c(), out.c()
        self._chk(self.L_.ckks_mul_relin_rescale(self.h, ctypes.byref(ca), ctypes.byref(cb), ctypes.byref(co)),
                  "ckks_mul_relin_rescale")
        return out.sync(co)

    def rescale(self, ct: Buf, out=None):
        out = self._out(ct, out, level=max(ct.level - 1, 1))
        ca, co = ct.c(), out.c()
        self._chk(self.L_.ckks_rescale(self.h, ctypes.byref(ca), ctypes.byref(co)), "ckks_rescale")
        return out.sync(co)

    def rotate(self, ct: Buf, steps: int, out=None):
        out = self._out(ct, out)
        ca, co = ct.c(), out.c()
        self._chk(self.L_.ckks_rotate(self.h, ctypes.byref(ca), steps, ctypes.byref(co)), "ckks_rotate")
        return out.sync(co)

    def total_sum(self, ct: Buf, out=None):
        out = self._out(ct, out)
        ca, co = ct.c(), out.c()
        self._chk(self.L_.ckks_total_sum(self.h, ctypes.byref(ca), ctypes.byref(co)), "ckks_total_sum")
        return out.sync(co)

    def modadd_gathered(self, gathered: torch.Tensor, R: int, out: Buf):
        co = out.c()
        self._chk(self.L_.ckks_modadd_gathered(self.h, _ptr(gathered), R, ctypes.byref(co)), "ckks_modadd_gathered")
        return out

    # ---- limb-sharded key switching --------------------------------------------
    def shard_ks_digits(self, kind: int, step: int, a: Buf, b: Buf | None, lo: int, l: int, w: int,
                        out: Buf | None, D_own: torch.Tensor):
        ca = a.c()
        cb = b.c() if b is not None else None
        co = out.c() if out is not None else None
        self._chk(self.L_.ckks_shard_ks_digits(self.h, kind, step, ctypes.byref(ca),
                                               ctypes.byref(cb) if cb is not None else None, lo, l, w,
                                               ctypes.byref(co) if co is not None else None, _ptr(D_own)),
                  "ckks_shard_ks_digits")
        if out is not None:
            out.sync(co)
        return out

    def shard_ks_finish(self, kind: int, step: int, D_all: torch.Tensor, R: int, w: int, a: Buf, lo: int, l: int,
                        out: Buf):
        ca, co = a.c(), out.c()
        self._chk(self.L_.ckks_shard_ks_finish(self.h, kind, step, _ptr(D_all), R, w, ctypes.byref(ca), lo, l,
                                               ctypes.byref(co)), "ckks_shard_ks_finish")
        return out.sync(co)

    def shard_ks_window(self, kind: int, step: int, D_win: torch.Tensor, r: int, w: int, a: Buf, lo: int, l: int,
                        first: bool):
        ca = a.c()
        self._chk(self.L_.ckks_shard_ks_window(self.h, kind, step, _ptr(D_win), r, w, ctypes.byref(ca), lo, l,
                                               int(first)), "ckks_shard_ks_window")

    def shard_ks_combine(self, kind: int, step: int, a: Buf, lo: int, l: int, out: Buf) -> Buf:
        ca, co = a.c(), out.c()
        self._chk(self.L_.ckks_shard_ks_combine(self.h, kind, step, ctypes.byref(ca), lo, l, ctypes.byref(co)),
                  "ckks_shard_ks_combine")
        return out.sync(co)

    def shard_rescale_last(self, ct: Buf, lo: int, l: int, X: torch.Tensor):
        cc = ct.c()
        self._chk(self.L_.ckks_shard_rescale_last(self.h, ctypes.byref(cc), lo, l, _ptr(X)), "ckks_shard_rescale_last")

    def shard_rescale_apply(self, X: torch.Tensor, ct: Buf, lo: int, l: int, out: Buf):
        cc, co = ct.c(), out.c()
        self._chk(self.L_.ckks_shard_rescale_apply(self.h, _ptr(X), ctypes.byref(cc), lo, l, ctypes.byref(co)),
                  "ckks_shard_rescale_apply")
        return out.sync(co)

    # ---- PrivFT ----------------------------------------------------------------------------
    def privft_model_create(self, H: np.ndarray, O: np.ndarray) -> "Model":
        H = np.ascontiguousarray(H, dtype=np.float64)
        O = np.ascontiguousarray(O, dtype=np.float64)
        h = c_vp()
        self._chk(self.L_.ckks_privft_model_create(self.h, H.ctypes.data_as(P(c_dbl)), O.ctypes.data_as(P(c_dbl)),
                                                   H.shape[0], H.shape[1], O.shape[1], ctypes.byref(h)),
                  "ckks_privft_model_create")
        return Model(self, h, None, n=H.shape[1], K=-(-H.shape[0] // (self.N // 2)))

    def privft_model_wrap(self, H_pts: Buf, O_pts: Buf, m: int, n: int, c: int) -> "Model":
        h = c_vp()
        hb, ob = H_pts.c(), O_pts.c()
        self._chk(self.L_.ckks_privft_model_wrap(self.h, ctypes.byref(hb), ctypes.byref(ob), m, n, c, ctypes.byref(h)),
                  "ckks_privft_model_wrap")
        return Model(self, h, (H_pts, O_pts), n=n, K=-(-m // (self.N // 2)))

    def privft_chunkdot(self, model: "Model", bag: Buf, out: Buf | None = None) -> Buf:
        """v.H alone: count batch*n ciphertexts at level L, no rescale."""
        batch = bag.count // model.K
        out = out if out is not None else self.alloc(batch * model.n, 2, self.L, None, 1.0)
        cb, ob = bag.c(), out.c()
        self._chk(self.L_.ckks_privft_chunkdot(self.h, model.h, ctypes.byref(cb), batch, ctypes.byref(ob)),
                  "ckks_privft_chunkdot")
        return out.sync(ob)

    def privft_infer(self, model: "Model", bag: Buf, w, poly_softmax: bool, out: Buf | None = None) -> Buf:
        w = np.ascontiguousarray(np.asarray(w, dtype=np.uint32))
        batch = w.size
        if out is None:
            out = self.alloc(batch, 2, self.L - 3, self.L - 3, 1.0)
        cb, co = bag.c(), out.c()
        self._chk(self.L_.ckks_privft_infer(self.h, model.h, ctypes.byref(cb), w.ctypes.data_as(P(c_u32)), batch,
                                            POLY_SOFTMAX if poly_softmax else 0, ctypes.byref(co)),
                  "ckks_privft_infer")
        return out.sync(co)

    def privft_infer_host(self, model: "Model", bag_host: torch.Tensor, bag_scale: float, w, poly_softmax: bool,
                          scores_host: torch.Tensor):
        """ckks_privft_infer_host: bag and scores in (pinned) HOST int64 tensors; asynchronous --
        call sync() before reading scores_host.  Returns (scores scale, scores level)."""
        assert not bag_host.is_cuda and not scores_host.is_cuda and bag_host.is_contiguous()
        w = np.ascontiguousarray(np.asarray(w, dtype=np.uint32))
        # Host memory must outlive the enqueued copies.  The library alternates two staging
        # slots per call and call k's copies may still be queued when call k+1 returns, so
        # keep one reference set per slot (released by sync()).
        slot = self._host_calls & 1
        self._host_calls += 1
        self._keep[slot] = (w, bag_host, scores_host)
        sc, lv = c_dbl(), c_u32()
        self._chk(self.L_.ckks_privft_infer_host(self.h, model.h, c_vp(bag_host.data_ptr()), bag_scale,
                                                 w.ctypes.data_as(P(c_u32)), w.size,
                                                 POLY_SOFTMAX if poly_softmax else 0, c_vp(scores_host.data_ptr()),
                                                 ctypes.byref(sc), ctypes.byref(lv)), "ckks_privft_infer_host")
        return sc.value, lv.value

    def sync(self):
        self._chk(self.L_.ckks_sync(self.h), "ckks_sync")
        self._keep = [None, None]


def _train_methods():
    def privft_train_plan(self, H: Buf, O: Buf, bags: Buf):
        """(scale, level) at which -onehot and the class mask must be encoded."""
        sc, lv = c_dbl(), c_u32()
        ch, co, cb = H.c(), O.c(), bags.c()
        self._chk(self.L_.ckks_privft_train_plan(self.h, ctypes.byref(ch), ctypes.byref(co), ctypes.byref(cb),
                                                 ctypes.byref(sc), ctypes.byref(lv)), "ckks_privft_train_plan")
        return sc.value, lv.value

    def privft_train_grad(self, H: Buf, O: Buf, bags: Buf, w, y, n_classes: int, neg_onehot: Buf, mask: Buf):
        """Encrypted gradient sums (GH at level l0-8, GO at level l0-6) over a minibatch."""
        w = np.ascontiguousarray(np.asarray(w, dtype=np.uint32))
        y = np.ascontiguousarray(np.asarray(y, dtype=np.uint32))
        GH = self.alloc(H.count, 2, H.level - 8)
        GO = self.alloc(H.count, 2, H.level - 6)
        ch, co, cb, cgh, cgo = H.c(), O.c(), bags.c(), GH.c(), GO.c()
        coh, cm = neg_onehot.c(), mask.c()
        self._chk(self.L_.ckks_privft_train_grad(self.h, ctypes.byref(ch), ctypes.byref(co), ctypes.byref(cb),
                                                 w.ctypes.data_as(P(c_u32)), y.ctypes.data_as(P(c_u32)), n_classes,
                                                 ctypes.byref(coh), ctypes.byref(cm), ctypes.byref(cgh),
                                                 ctypes.byref(cgo)), "ckks_privft_train_grad")
        return GH.sync(cgh), GO.sync(cgo)

    def privft_train_update(self, H: Buf, O: Buf, GH: Buf, GO: Buf, eta: float):
        """(H - eta GH, O - eta GO), both at level l0 - 9."""
        Hn = self.alloc(H.count, 2, H.level - 9)
        On = self.alloc(O.count, 2, O.level - 9)
        ch, co, cgh, cgo, chn, con = H.c(), O.c(), GH.c(), GO.c(), Hn.c(), On.c()
        self._chk(self.L_.ckks_privft_train_update(self.h, ctypes.byref(ch), ctypes.byref(co), ctypes.byref(cgh),
                                                   ctypes.byref(cgo), eta, ctypes.byref(chn), ctypes.byref(con)),
                  "ckks_privft_train_update")
        return Hn.sync(chn), On.sync(con)

    Context.privft_train_plan = privft_train_plan
    Context.privft_train_grad = privft_train_grad
    Context.privft_train_update = privft_train_update


_train_methods()


class Model:
    def __init__(self, ctx: Context, h, keepalive, n: int = 0, K: int = 0):
        self.ctx, self.h, self._keep = ctx, h, keepalive
        self.n, self.K = n, K  # embedding dimension, chunks per query

    def __del__(self):
        try:
            if self.h:
                self.ctx.L_.ckks_privft_model_destroy(self.h)
        except Exception:
            pass
