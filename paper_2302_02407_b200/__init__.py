"""paper_2302_02407_b200 -- B200-native HyPHEN homomorphic-convolution hot path.

Thin Python binding over the C ABI of ``libhyphen.so`` (declared in
``include/hyphen.h``).  Argument marshalling only: every step of the path runs
in the library's sm_100a kernels.  PyTorch provides device memory (int64
tensors holding the uint64 residues bit-for-bit), streams and process groups.
There is no CPU fallback: when the library or a CUDA device is missing, the
calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhyphen.so")

HY_ERRORS = {
    0: "HY_OK", 1: "HY_E_ARG", 2: "HY_E_LEVEL_MISMATCH", 3: "HY_E_LEVEL_EXHAUSTED", 4: "HY_E_SHAPE",
    5: "HY_E_CAPACITY", 6: "HY_E_FORMAT", 7: "HY_E_PLAN", 8: "HY_E_MISSING_KEY", 9: "HY_E_CUDA",
    10: "HY_E_WORKSPACE", 11: "HY_E_NO_DEVICE",
}


class HyError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{HY_ERRORS.get(code, code)}: {msg}")
        self.code = code


class _Params(C.Structure):
    _fields_ = [("log_n", C.c_uint32), ("n_q", C.c_uint32), ("n_p", C.c_uint32), ("dnum", C.c_uint32),
                ("hamming_weight", C.c_uint32), ("q_bits", C.POINTER(C.c_uint32)), ("p_bits", C.POINTER(C.c_uint32))]


class _ConvSpec(C.Structure):
    _fields_ = [(k, C.c_uint32) for k in ("ci", "co", "w", "f", "stride", "wp", "gap", "m", "d", "algo",
                                          "segments", "bias")]


_lib = None
_P = C.c_void_p
_U64 = C.c_uint64
_U32 = C.c_uint32
_PP = C.POINTER(C.c_void_p)

SIGNATURES = {
    "hy_ctx_create": (C.c_int, [C.POINTER(_Params), C.c_int, C.POINTER(_P)]),
    "hy_ctx_destroy": (None, [_P]),
    "hy_ctx_moduli": (C.c_int, [_P, C.POINTER(_U64)]),
    "hy_ctx_alpha": (_U32, [_P]),
    "hy_ctx_n_digits": (_U32, [_P, _U32]),
    "hy_workspace_bytes": (C.c_size_t, [_P, _U32, _U32]),
    "hy_ctx_set_workspace": (C.c_int, [_P, _P, C.c_size_t]),
    "hy_last_error": (C.c_char_p, []),
    "hy_ctx_launch_count": (_U64, [_P]),
    "hy_ctx_time_kernels": (C.c_int, [_P, _U32]),
    "hy_ctx_kernel_times": (C.c_int, [_P, _U32, C.POINTER(C.c_double), C.POINTER(_U64), C.POINTER(_U64)]),
    "hy_ntt": (C.c_int, [_P, _P, _P, C.POINTER(_U32), _U32, C.c_int, _P]),
    "hy_automorph": (C.c_int, [_P, _P, _P, _U32, _U64, _P]),
    "hy_galois_elt": (_U64, [_P, C.c_int64]),
    "hy_prot": (C.c_int, [_P, _P, _U32, C.c_int32, _P, _P]),
    "hy_modup": (C.c_int, [_P, _U32, _P, _P, _P]),
    "hy_ks_inner_product": (C.c_int, [_P, _U32, _P, _P, _P, _P]),
    "hy_moddown": (C.c_int, [_P, _U32, _P, _P, _P]),
    "hy_hrot": (C.c_int, [_P, _P, _P, _U32, C.c_int32, _P, _P]),
    "hy_hrot_batch": (C.c_int, [_P, _PP, _PP, _U32, C.POINTER(C.c_int32), _U32, _PP, _P]),
    "hy_hrot_hoisted": (C.c_int, [_P, _PP, _P, _U32, C.POINTER(C.c_int32), _U32, _PP, _P]),
    "hy_hrot_sum": (C.c_int, [_P, _PP, _PP, _U32, C.POINTER(C.c_int32), _U32, _P, _P]),
    "hy_pmult": (C.c_int, [_P, _P, _P, _U32, _P, _P]),
    "hy_pmult_acc": (C.c_int, [_P, _PP, _PP, _U32, _U32, _P, C.c_int, _P]),
    "hy_add": (C.c_int, [_P, _P, _P, _U32, _U32, _P, _P]),
    "hy_rescale": (C.c_int, [_P, _P, _U32, _P, _P]),
    "hy_level_down": (C.c_int, [_P, _P, _U32, _U32, _P, _P]),
    "hy_keygen_rot": (C.c_int, [_P, _U64, _U64, C.c_int32, _P, _P]),
    "hy_keygen_galois": (C.c_int, [_P, _U64, _U64, _U64, _P, _P]),
    "hy_keygen_relin": (C.c_int, [_P, _U64, _U64, _P, _P]),
    "hy_evk_words": (C.c_size_t, [_P]),
    "hy_evk_pack": (C.c_int, [_P, _P, _P, _P]),
    "hy_evk_unpack": (C.c_int, [_P, _P, _P, _P]),
    "hy_pack48": (C.c_int, [_P, _P, _P, C.c_size_t, _P]),
    "hy_unpack48": (C.c_int, [_P, _P, _P, C.c_size_t, _P]),
    "hy_mulct": (C.c_int, [_P, _P, _P, _P, _U32, _P, _P]),
    "hy_mulct_batch": (C.c_int, [_P, _P, _PP, _PP, _U32, _U32, _PP, _P]),
    "hy_rescale_batch": (C.c_int, [_P, _PP, _U32, _U32, _PP, _P]),
    "hy_pmult_batch": (C.c_int, [_P, _PP, _U32, _P, _U32, _PP, _P]),
    "hy_encrypt": (C.c_int, [_P, _U64, _U64, _U64, _P, _U32, _P, _P]),
    "hy_decrypt": (C.c_int, [_P, _U64, _P, _U32, _P, _P]),
    "hy_encode": (C.c_int, [_P, C.POINTER(C.c_double), _U32, _U64, _U32, _P, _P]),
    "hy_encode_coeffs": (C.c_int, [_U32, C.POINTER(C.c_double), _U32, _U64, C.POINTER(C.c_int64)]),
    "hy_pt_from_coeffs": (C.c_int, [_P, C.POINTER(C.c_int64), _U32, _P, _P]),
    "hy_encode_batch": (C.c_int, [_P, C.POINTER(C.c_double), _U32, _U64, _U32, _P, _P]),
    "hy_decode": (C.c_int, [_P, _P, _U32, C.c_double, _U32, C.POINTER(C.c_double), C.POINTER(C.c_double), _P]),
    "hy_decode_coeffs": (C.c_int, [_U32, C.POINTER(C.c_double), C.c_double, _U32, C.POINTER(C.c_double),
                                   C.POINTER(C.c_double)]),
    "hy_conv_plan_create": (C.c_int, [_U32, C.POINTER(_ConvSpec), C.POINTER(_P)]),
    "hy_conv_plan_destroy": (None, [_P]),
    "hy_conv_plan_query": (C.c_int, [_P, C.POINTER(_U32), C.POINTER(_U32), C.POINTER(_U32), C.POINTER(_U32),
                                      C.POINTER(_U32), C.POINTER(C.c_int32), C.POINTER(_U32)]),
    "hy_conv_weight_slots": (C.c_int, [_P, C.POINTER(C.c_double), _U32, C.POINTER(C.c_double)]),
    "hy_conv_weight_words": (C.c_size_t, [_P, _P, _U32]),
    "hy_conv_scratch_words": (C.c_size_t, [_P, _P, _U32]),
    "hy_conv_encode_weights": (C.c_int, [_P, _P, C.POINTER(C.c_double), C.POINTER(C.c_double), _U64, _U32, _P,
                                         _P]),
    "hy_conv_bias_slots": (C.c_int, [_P, C.POINTER(C.c_double), _U32, C.POINTER(C.c_double)]),
    "hy_encode_coeffs_complex": (C.c_int, [_U32, C.POINTER(C.c_double), C.POINTER(C.c_double), _U32, _U64,
                                           C.POINTER(C.c_int64)]),
    "hy_mod_raise": (C.c_int, [_P, _P, _U32, _P, _P]),
    "hy_sub": (C.c_int, [_P, _P, _P, _U32, _U32, _P, _P]),
    "hy_hrot_galois": (C.c_int, [_P, _P, _P, _U32, _U64, _P, _P]),
    "hy_lintrans_create": (C.c_int, [_U32, C.POINTER(C.c_int32), _U32, _U32, C.POINTER(_P)]),
    "hy_lintrans_destroy": (None, [_P]),
    "hy_lintrans_query": (C.c_int, [_P, C.POINTER(_U32), C.POINTER(_U32), C.POINTER(_U32), C.POINTER(_U32),
                                     C.POINTER(C.c_int32)]),
    "hy_lintrans_pt_words": (C.c_size_t, [_P, _P, _U32]),
    "hy_lintrans_scratch_words": (C.c_size_t, [_P, _P, _U32]),
    "hy_lintrans_encode": (C.c_int, [_P, _P, C.POINTER(C.c_double), C.POINTER(C.c_double), _U32, _P, _P]),
    "hy_lintrans_apply": (C.c_int, [_P, _P, _PP, _P, _U32, _P, _P, _P, _P]),
    "hy_keyset_create": (C.c_int, [_U32, C.POINTER(C.c_int32), _U32, C.POINTER(_P)]),
    "hy_keyset_destroy": (None, [_P]),
    "hy_keyset_decompose": (C.c_int, [_P, C.c_int32, C.POINTER(C.c_int32), _U32, C.POINTER(_U32)]),
    "hy_conv_plan_set_keyset": (C.c_int, [_P, _P]),
    "hy_conv_plan_eff_counts": (C.c_int, [_P, C.POINTER(_U32)]),
    "hy_add_pt": (C.c_int, [_P, _P, C.c_double, _P, C.c_double, _U32, _P, _P]),
    "hy_ct_bytes": (C.c_size_t, [_P, _U32]),
    "hy_pt_bytes": (C.c_size_t, [_P, _U32, C.c_int]),
    "hy_export_coeff": (C.c_int, [_P, _P, C.POINTER(_U32), _U32, C.POINTER(_U64), _P]),
    "hy_import_coeff": (C.c_int, [_P, C.POINTER(_U64), C.POINTER(_U32), _U32, _P, _P]),
    "hy_caconv": (C.c_int, [_P, _P, _PP, _PP, _U32, _P, _P, _U32, _U32, _PP, _P]),
    "hy_raconv": (C.c_int, [_P, _P, _PP, _PP, _U32, _P, _P, _U32, _U32, _PP, _P]),
    "hy_caconv_slide": (C.c_int, [_P, _P, _PP, _PP, _U32, _U32, _U32, _P, _P]),
    "hy_caconv_slid": (C.c_int, [_P, _P, _PP, _P, _U32, _P, _P, _U32, _U32, _PP, _P]),
    "hy_raconv_partial_words": (C.c_size_t, [_P, _U32]),
    "hy_raconv_partial": (C.c_int, [_P, _P, _PP, _PP, _U32, _P, _P, _U32, _U32, _U32, _P, _P]),
    "hy_raconv_finish": (C.c_int, [_P, _P, _PP, _U32, _P, _P, _P, _U32, _P, _P]),
}


def lib():
    """Load libhyphen.so (raises if it was not built: no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -m paper_2302_02407_b200.build` "
                              "(or __graft_entry__.build()); there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(code: int):
    if code != 0:
        raise HyError(code, lib().hy_last_error().decode())


def _ptr(t) -> int:
    return t.data_ptr() if t is not None else 0


def _ptr_array(ts):
    a = (C.c_void_p * max(1, len(ts)))()
    for i, t in enumerate(ts):
        a[i] = _ptr(t)
    return a


def encode_coeffs(log_n: int, slots, scale: int) -> np.ndarray:
    """Host-side CKKS encoding (DESIGN R-ENCODE): N signed integer coefficients."""
    z = np.ascontiguousarray(slots, np.float64)
    out = np.zeros(1 << log_n, np.int64)
    _check(lib().hy_encode_coeffs(log_n, z.ctypes.data_as(C.POINTER(C.c_double)), len(z), int(scale),
                                  out.ctypes.data_as(C.POINTER(C.c_int64))))
    return out


def decode_coeffs(log_n: int, coeffs, scale: float, n_slots=None) -> np.ndarray:
    """Host-side CKKS decoding of real coefficients: complex slots z_j = m(zeta^{5^j}) / scale."""
    m = np.ascontiguousarray(coeffs, np.float64)
    n_slots = (1 << log_n) // 2 if n_slots is None else n_slots
    re, im = np.zeros(n_slots), np.zeros(n_slots)
    _check(lib().hy_decode_coeffs(log_n, m.ctypes.data_as(C.POINTER(C.c_double)), float(scale), n_slots,
                                  re.ctypes.data_as(C.POINTER(C.c_double)), im.ctypes.data_as(C.POINTER(C.c_double))))
    return re + 1j * im


class Context:
    """One RNS-CKKS context on one CUDA device (see include/hyphen.h)."""

    def __init__(self, log_n, q_bits, p_bits, dnum, h=192, device=0, max_level=None, max_batch=None, **_):
        import torch

        self.torch = torch
        self.device = torch.device("cuda", device)
        self.log_n, self.N, self.n = log_n, 1 << log_n, 1 << (log_n - 1)
        self.n_q, self.n_p, self.dnum, self.h = len(q_bits), len(p_bits), dnum, h
        self._qb = (C.c_uint32 * len(q_bits))(*q_bits)
        self._pb = (C.c_uint32 * len(p_bits))(*p_bits)
        prm = _Params(log_n, len(q_bits), len(p_bits), dnum, h, self._qb, self._pb)
        h_ = C.c_void_p()
        self._lib = lib()
        _check(self._lib.hy_ctx_create(C.byref(prm), device, C.byref(h_)))
        self._c = h_
        mods = (C.c_uint64 * (self.n_q + self.n_p))()
        _check(lib().hy_ctx_moduli(self._c, mods))
        self.moduli = [int(x) for x in mods]
        self.q, self.p = self.moduli[: self.n_q], self.moduli[self.n_q:]
        self.alpha = int(lib().hy_ctx_alpha(self._c))
        self.max_level = self.n_q - 1 if max_level is None else max_level
        # workspace for up to `max_batch` key switches per batched launch (library cap: 64; HY_MAX_BATCH)
        if max_batch is None:
            max_batch = int(os.environ.get("HY_MAX_BATCH", "16"))
        nbytes = int(lib().hy_workspace_bytes(self._c, self.max_level, max_batch))
        self.ws = torch.empty(nbytes // 8 + 1, dtype=torch.int64, device=self.device)
        _check(lib().hy_ctx_set_workspace(self._c, self.ws.data_ptr(), self.ws.numel() * 8))

    def __del__(self):
        # the library handle is held by the object: module globals may be gone at interpreter exit
        if getattr(self, "_c", None) and getattr(self, "_lib", None) is not None:
            self._lib.hy_ctx_destroy(self._c)
            self._c = None

    # -- helpers ---------------------------------------------------------
    def _stream(self):
        return C.c_void_p(self.torch.cuda.current_stream(self.device).cuda_stream)

    def empty(self, *shape):
        return self.torch.empty(*shape, dtype=self.torch.int64, device=self.device)

    def zeros(self, *shape):
        return self.torch.zeros(*shape, dtype=self.torch.int64, device=self.device)

    def ct_shape(self, level):
        return (2, level + 1, self.N)

    def evk_shape(self):
        """packed key (include/hyphen.h Conventions): 6 bytes per word, 3N/4 uint64 per limb"""
        return (self.dnum, 2, self.n_q + self.n_p, self.N // 4 * 3)

    def evk_bytes(self):
        """bytes of one packed evaluation key at full level (126 MiB at Set_hyp; 168 MB unpacked)"""
        return int(lib().hy_evk_words(self._c)) * 8

    def evk_pack(self, evk_u64, out=None):
        """[dnum][2][n_q+n_p][N] one word per uint64 (e.g. the oracle's key) -> packed device key"""
        out = self.empty(*self.evk_shape()) if out is None else out
        _check(lib().hy_evk_pack(self._c, _ptr(evk_u64), _ptr(out), self._stream()))
        return out

    def pack48(self, t, out=None):
        """residue tensor (numel % 4 == 0) -> 48-bit wire format, 3 numel / 4 int64 words (hy_pack48)"""
        out = self.empty(t.numel() // 4 * 3) if out is None else out
        _check(lib().hy_pack48(self._c, _ptr(t), _ptr(out), t.numel(), self._stream()))
        return out

    def unpack48(self, packed, out):
        """48-bit wire format -> residues into `out` (its numel words, hy_unpack48)"""
        _check(lib().hy_unpack48(self._c, _ptr(packed), _ptr(out), out.numel(), self._stream()))
        return out

    def evk_unpack(self, evk, out=None):
        out = self.empty(self.dnum, 2, self.n_q + self.n_p, self.N) if out is None else out
        _check(lib().hy_evk_unpack(self._c, _ptr(evk), _ptr(out), self._stream()))
        return out

    def n_digits(self, level):
        return int(lib().hy_ctx_n_digits(self._c, level))

    def galois_elt(self, r: int) -> int:
        return int(lib().hy_galois_elt(self._c, int(r)))

    def launch_count(self) -> int:
        return int(lib().hy_ctx_launch_count(self._c))

    FAMILIES = {"ntt_a": 1, "ntt_b": 2, "modup": 4, "ip": 8, "moddown": 16, "aut": 32, "elem": 64,
                "rescale": 128, "client": 256, "ntt_ip": 512}

    def time_kernels(self, mask: int):
        _check(lib().hy_ctx_time_kernels(self._c, mask))

    def kernel_times(self, mask: int):
        """(total device ms, launches, algorithmic bytes) of the timed launches in `mask`."""
        ms, n, by = C.c_double(), C.c_uint64(), C.c_uint64()
        _check(lib().hy_ctx_kernel_times(self._c, mask, C.byref(ms), C.byref(n), C.byref(by)))
        return ms.value, n.value, by.value

    # -- transforms ------------------------------------------------------
    def ntt(self, x, chain: Sequence[int], inverse=False, out=None):
        out = self.empty(*x.shape) if out is None else out
        ch = (C.c_uint32 * len(chain))(*chain)
        _check(lib().hy_ntt(self._c, _ptr(x), _ptr(out), ch, len(chain), int(inverse), self._stream()))
        return out

    def automorph(self, x, k: int, out=None):
        out = self.empty(*x.shape) if out is None else out
        nl = x.numel() // self.N
        _check(lib().hy_automorph(self._c, _ptr(x), _ptr(out), nl, int(k), self._stream()))
        return out

    # -- key switching ---------------------------------------------------
    def prot(self, pt, level, r, out=None):
        """PRot: plaintext rotation by r slots (hy_prot)"""
        out = self.empty(level + 1, self.N) if out is None else out
        _check(lib().hy_prot(self._c, _ptr(pt), level, int(r), _ptr(out), self._stream()))
        return out

    def modup(self, level, d_coeff):
        ext = self.empty(self.n_digits(level), level + 1 + self.n_p, self.N)
        _check(lib().hy_modup(self._c, level, _ptr(d_coeff), _ptr(ext), self._stream()))
        return ext

    def ks_inner_product(self, level, ext, evk):
        u = self.empty(2, level + 1 + self.n_p, self.N)
        _check(lib().hy_ks_inner_product(self._c, level, _ptr(ext), _ptr(evk), _ptr(u), self._stream()))
        return u

    def moddown(self, level, u_poly):
        out = self.empty(level + 1, self.N)
        _check(lib().hy_moddown(self._c, level, _ptr(u_poly), _ptr(out), self._stream()))
        return out

    def hrot(self, evk, ct, level, r, out=None):
        out = self.empty(*self.ct_shape(level)) if out is None else out
        _check(lib().hy_hrot(self._c, _ptr(evk), _ptr(ct), level, int(r), _ptr(out), self._stream()))
        return out

    def hrot_batch(self, evks, cts, level, rs, outs=None):
        outs = [self.empty(*self.ct_shape(level)) for _ in cts] if outs is None else outs
        r = (C.c_int32 * len(rs))(*rs)
        _check(lib().hy_hrot_batch(self._c, _ptr_array(evks), _ptr_array(cts), level, r, len(rs),
                                   _ptr_array(outs), self._stream()))
        return outs

    def hrot_hoisted(self, evks, ct, level, rs, outs=None):
        outs = [self.empty(*self.ct_shape(level)) for _ in rs] if outs is None else outs
        r = (C.c_int32 * len(rs))(*rs)
        _check(lib().hy_hrot_hoisted(self._c, _ptr_array(evks), _ptr(ct), level, r, len(rs),
                                     _ptr_array(outs), self._stream()))
        return outs

    def hrot_sum(self, evks, cts, level, rs, out=None):
        out = self.empty(*self.ct_shape(level)) if out is None else out
        r = (C.c_int32 * len(rs))(*rs)
        _check(lib().hy_hrot_sum(self._c, _ptr_array(evks), _ptr_array(cts), level, r, len(rs), _ptr(out),
                                 self._stream()))
        return out

    # -- MulPt / AddCt / Rescale -----------------------------------------
    def pmult(self, ct, pt, level, out=None):
        out = self.empty(*self.ct_shape(level)) if out is None else out
        _check(lib().hy_pmult(self._c, _ptr(ct), _ptr(pt), level, _ptr(out), self._stream()))
        return out

    def pmult_acc(self, cts, pts, level, out=None, accumulate=False):
        out = self.empty(*self.ct_shape(level)) if out is None else out
        _check(lib().hy_pmult_acc(self._c, _ptr_array(cts), _ptr_array(pts), len(cts), level, _ptr(out),
                                  int(accumulate), self._stream()))
        return out

    def add(self, a, b, level, out=None, npoly=2):
        out = self.empty(*a.shape) if out is None else out
        _check(lib().hy_add(self._c, _ptr(a), _ptr(b), npoly, level, _ptr(out), self._stream()))
        return out

    def level_down(self, ct, level, new_level, out=None):
        out = self.empty(*self.ct_shape(new_level)) if out is None else out
        _check(lib().hy_level_down(self._c, _ptr(ct), level, new_level, _ptr(out), self._stream()))
        return out

    def rescale(self, ct, level, out=None):
        out = self.empty(*self.ct_shape(level - 1)) if out is None else out
        _check(lib().hy_rescale(self._c, _ptr(ct), level, _ptr(out), self._stream()))
        return out

    def pmult_batch(self, cts, pt, level, outs=None):
        """ct_i (.) pt for every ciphertext, one plaintext, one launch (hy_pmult_batch)"""
        outs = [self.empty(*self.ct_shape(level)) for _ in cts] if outs is None else outs
        _check(lib().hy_pmult_batch(self._c, _ptr_array(cts), len(cts), _ptr(pt), level, _ptr_array(outs),
                                    self._stream()))
        return outs

    def rescale_batch(self, cts, level, outs=None):
        outs = [self.empty(*self.ct_shape(level - 1)) for _ in cts] if outs is None else outs
        _check(lib().hy_rescale_batch(self._c, _ptr_array(cts), len(cts), level, _ptr_array(outs), self._stream()))
        return outs

    # -- client side -----------------------------------------------------
    def keygen_rot(self, sk_seed, ek_seed, r, out=None):
        out = self.empty(*self.evk_shape()) if out is None else out
        _check(lib().hy_keygen_rot(self._c, sk_seed, ek_seed, int(r), _ptr(out), self._stream()))
        return out

    def keygen_relin(self, sk_seed, ek_seed, out=None):
        out = self.empty(*self.evk_shape()) if out is None else out
        _check(lib().hy_keygen_relin(self._c, sk_seed, ek_seed, _ptr(out), self._stream()))
        return out

    def mulct(self, rlk, a, b, level, out=None):
        """MulCt + relinearization, no rescale (include/hyphen.h hy_mulct)."""
        out = self.empty(*self.ct_shape(level)) if out is None else out
        _check(lib().hy_mulct(self._c, _ptr(rlk), _ptr(a), _ptr(b), level, _ptr(out), self._stream()))
        return out

    def mulct_batch(self, rlk, As, Bs, level, outs=None):
        """a_i * b_i for every pair, MulCt + relinearization in one batched key switch, no rescale (hy_mulct_batch)."""
        outs = [self.empty(*self.ct_shape(level)) for _ in As] if outs is None else outs
        _check(lib().hy_mulct_batch(self._c, _ptr(rlk), _ptr_array(As), _ptr_array(Bs), level, len(As),
                                    _ptr_array(outs), self._stream()))
        return outs

    def square_batch(self, rlk, cts, level, outs=None):
        """x^2 of every ciphertext (AESPA after fusion), MulCt + relinearization, no rescale."""
        outs = [self.empty(*self.ct_shape(level)) for _ in cts] if outs is None else outs
        _check(lib().hy_mulct_batch(self._c, _ptr(rlk), _ptr_array(cts), _ptr_array(cts), level, len(cts),
                                    _ptr_array(outs), self._stream()))
        return outs

    def keygen_galois(self, sk_seed, ek_seed, k, out=None):
        out = self.empty(*self.evk_shape()) if out is None else out
        _check(lib().hy_keygen_galois(self._c, sk_seed, ek_seed, int(k), _ptr(out), self._stream()))
        return out

    def encrypt(self, sk_seed, enc_seed, ct_id, pt, level, out=None):
        out = self.empty(*self.ct_shape(level)) if out is None else out
        _check(lib().hy_encrypt(self._c, sk_seed, enc_seed, ct_id, _ptr(pt), level, _ptr(out), self._stream()))
        return out

    def decrypt(self, sk_seed, ct, level, out=None):
        out = self.empty(level + 1, self.N) if out is None else out
        _check(lib().hy_decrypt(self._c, sk_seed, _ptr(ct), level, _ptr(out), self._stream()))
        return out

    def encode(self, slots, scale, level, out=None):
        out = self.empty(level + 1, self.N) if out is None else out
        z = np.ascontiguousarray(slots, np.float64)
        _check(lib().hy_encode(self._c, z.ctypes.data_as(C.POINTER(C.c_double)), len(z), int(scale), level,
                               _ptr(out), self._stream()))
        return out

    def encode_batch(self, slots, scale, level, out=None):
        """P real slot vectors [P][N/2] -> [P][level+1][N] plaintexts, encoded on the device (hy_encode_batch)"""
        z = np.ascontiguousarray(slots, np.float64).reshape(-1, self.n)
        out = self.empty(z.shape[0], level + 1, self.N) if out is None else out
        _check(lib().hy_encode_batch(self._c, z.ctypes.data_as(C.POINTER(C.c_double)), z.shape[0], int(scale),
                                     level, _ptr(out), self._stream()))
        return out

    def decode(self, pt, level, scale, n_slots=None):
        """Complex slots of an NTT-domain plaintext (hy_decode; synchronous)."""
        n_slots = self.N // 2 if n_slots is None else n_slots
        re, im = np.zeros(n_slots), np.zeros(n_slots)
        _check(lib().hy_decode(self._c, _ptr(pt), level, float(scale), n_slots,
                               re.ctypes.data_as(C.POINTER(C.c_double)), im.ctypes.data_as(C.POINTER(C.c_double)),
                               self._stream()))
        return re + 1j * im

    def add_pt(self, ct, ct_scale, pt, pt_scale, level, out=None):
        """AddPt (hy_add_pt): (c0 + pt, c1); HY_E_SCALE_MISMATCH when the scales differ."""
        out = self.empty(*self.ct_shape(level)) if out is None else out
        _check(lib().hy_add_pt(self._c, _ptr(ct), float(ct_scale), _ptr(pt), float(pt_scale), level, _ptr(out),
                               self._stream()))
        return out

    def ct_bytes(self, level):
        return int(lib().hy_ct_bytes(self._c, level))

    def pt_bytes(self, level, with_p=False):
        return int(lib().hy_pt_bytes(self._c, level, int(with_p)))

    def export_coeff(self, x, chain):
        """NTT-domain device limbs [len(chain)][N] -> coefficient-domain host uint64 array (hy_export_coeff)"""
        ch = (_U32 * len(chain))(*chain)
        out = np.empty((len(chain), self.N), np.uint64)
        _check(lib().hy_export_coeff(self._c, _ptr(x), ch, len(chain), out.ctypes.data_as(C.POINTER(_U64)),
                                     self._stream()))
        return out

    def import_coeff(self, a, chain, out=None):
        """coefficient-domain host limbs -> NTT-domain device limbs (hy_import_coeff)"""
        a = np.ascontiguousarray(a, np.uint64).reshape(len(chain), self.N)
        ch = (_U32 * len(chain))(*chain)
        out = self.empty(len(chain), self.N) if out is None else out
        _check(lib().hy_import_coeff(self._c, a.ctypes.data_as(C.POINTER(_U64)), ch, len(chain), _ptr(out),
                                     self._stream()))
        return out

    def sub(self, a, b, level, out=None, npoly=2):
        out = self.empty(npoly, level + 1, self.N) if out is None else out
        _check(lib().hy_sub(self._c, _ptr(a), _ptr(b), npoly, level, _ptr(out), self._stream()))
        return out

    def hrot_galois(self, evk, ct, level, k, out=None):
        """key switch by Galois element k (hy_hrot_galois; k = 2N - 1: conjugation)"""
        out = self.empty(*self.ct_shape(level)) if out is None else out
        _check(lib().hy_hrot_galois(self._c, _ptr(evk), _ptr(ct), level, int(k), _ptr(out), self._stream()))
        return out

    def mod_raise(self, ct0, level, out=None):
        """ModRaise (hy_mod_raise): level-0 ciphertext -> level `level`"""
        out = self.empty(*self.ct_shape(level)) if out is None else out
        _check(lib().hy_mod_raise(self._c, _ptr(ct0), level, _ptr(out), self._stream()))
        return out

    def encode_complex(self, z, scale, level):
        """complex slots -> NTT-domain plaintext (hy_encode_coeffs_complex + hy_pt_from_coeffs)"""
        z = np.asarray(z, np.complex128)
        re, im = np.ascontiguousarray(z.real), np.ascontiguousarray(z.imag)
        cf = np.zeros(self.N, np.int64)
        _check(lib().hy_encode_coeffs_complex(self.log_n, re.ctypes.data_as(C.POINTER(C.c_double)),
                                              im.ctypes.data_as(C.POINTER(C.c_double)), len(z), int(scale),
                                              cf.ctypes.data_as(C.POINTER(C.c_int64))))
        return self.pt_from_coeffs(cf, level)

    def pt_from_coeffs(self, coeffs, level, out=None):
        out = self.empty(level + 1, self.N) if out is None else out
        cf = np.ascontiguousarray(coeffs, np.int64)
        _check(lib().hy_pt_from_coeffs(self._c, cf.ctypes.data_as(C.POINTER(C.c_int64)), level, _ptr(out),
                                       self._stream()))
        return out


class LinTrans:
    """Homomorphic diagonal linear transform y = M x (bootstrapping's CoeffToSlot / SlotToCoeff building block;
    include/hyphen.h hy_lintrans_*, DESIGN R-LINTRANS): diagonals `diags` (amounts mod n), baby-step size bs."""

    def __init__(self, ctx, diags, bs, log_n=None):
        self.ctx = ctx
        log_n = log_n if log_n is not None else ctx.log_n
        self.n = 1 << (log_n - 1)
        d = (C.c_int32 * len(diags))(*[int(x) for x in diags])
        h = C.c_void_p()
        self._lib = lib()
        _check(self._lib.hy_lintrans_create(log_n, d, len(diags), int(bs), C.byref(h)))
        self._p = h
        npt, nb, ng, nr = (C.c_uint32() for _ in range(4))
        _check(lib().hy_lintrans_query(self._p, C.byref(npt), C.byref(nb), C.byref(ng), C.byref(nr), None))
        rots = (C.c_int32 * max(1, nr.value))()
        _check(lib().hy_lintrans_query(self._p, None, None, None, None, rots))
        self.n_pt, self.n_baby, self.n_giant = npt.value, nb.value, ng.value
        self.rots = [int(rots[i]) for i in range(nr.value)]
        self.diags = sorted({int(x) % self.n for x in diags})

    def __del__(self):
        if getattr(self, "_p", None) and getattr(self, "_lib", None) is not None:
            self._lib.hy_lintrans_destroy(self._p)
            self._p = None

    def encode(self, diag_values, level):
        """diag_values: complex [len(diags)][n] in ascending canonical d order"""
        v = np.asarray(diag_values)
        re = np.ascontiguousarray(np.real(v), np.float64)
        im = np.ascontiguousarray(np.imag(v), np.float64)
        pts = self.ctx.empty(int(lib().hy_lintrans_pt_words(self.ctx._c, self._p, level)))
        _check(lib().hy_lintrans_encode(self.ctx._c, self._p, re.ctypes.data_as(C.POINTER(C.c_double)),
                                        im.ctypes.data_as(C.POINTER(C.c_double)), level, _ptr(pts),
                                        self.ctx._stream()))
        return pts

    def apply(self, evks, ct, level, pts, scratch=None, out=None):
        if isinstance(evks, dict):
            evks = [evks[r] for r in self.rots]
        out = self.ctx.empty(*self.ctx.ct_shape(level - 1)) if out is None else out
        scratch = self.ctx.empty(int(lib().hy_lintrans_scratch_words(self.ctx._c, self._p, level))) \
            if scratch is None else scratch
        _check(lib().hy_lintrans_apply(self.ctx._c, self._p, _ptr_array(evks), _ptr(ct), level, _ptr(pts),
                                       _ptr(scratch), _ptr(out), self.ctx._stream()))
        return out


class KeySet:
    """A limited set of loaded rotation keys (hy_keyset_create, DESIGN R-KEYSET); other amounts are synthesized
    as the shortest sums of loaded ones."""

    def __init__(self, log_n, amounts):
        self.n = 1 << (log_n - 1)
        a = (C.c_int32 * max(1, len(amounts)))(*[int(x) for x in amounts])
        h = C.c_void_p()
        self._lib = lib()
        _check(self._lib.hy_keyset_create(log_n, a, len(amounts), C.byref(h)))
        self._k = h

    def __del__(self):
        if getattr(self, "_k", None) and getattr(self, "_lib", None) is not None:
            self._lib.hy_keyset_destroy(self._k)
            self._k = None

    def decompose(self, r):
        n = C.c_uint32()
        _check(lib().hy_keyset_decompose(self._k, int(r), None, 0, C.byref(n)))
        st = (C.c_int32 * max(1, n.value))()
        _check(lib().hy_keyset_decompose(self._k, int(r), st, n.value, C.byref(n)))
        return [int(st[i]) for i in range(n.value)]


class ConvPlan:
    """A HyPHEN convolution layer (CAConv / RAConv_Reorder) on one context (include/hyphen.h)."""

    CA, RA = 0, 1

    def __init__(self, ctx, ci, co, w, f, stride, wp, gap, m, d, algo, log_n=None, S=1, bias=False):
        """ctx may be None (host-only plan inspection) when log_n is given.  bias: the layer adds a per-output-
        channel bias (AddPt after its last rescale, DESIGN R-BIAS)."""
        self.ctx = ctx
        self.n = 1 << ((log_n if log_n is not None else ctx.log_n) - 1)
        self.algo = {"CA": 0, "RA": 1}.get(algo, algo)
        self.bias = bool(bias)
        spec = _ConvSpec(ci, co, w, f, stride, wp, gap, m, d, self.algo, S, int(self.bias))
        h = C.c_void_p()
        self._lib = lib()
        _check(self._lib.hy_conv_plan_create(log_n if log_n is not None else ctx.log_n, C.byref(spec), C.byref(h)))
        self._p = h
        self._query()
        self.f = f

    def _query(self):
        ni, no, npt, hm, nr = (C.c_uint32() for _ in range(5))
        counts = (C.c_uint32 * 5)()
        _check(lib().hy_conv_plan_query(self._p, C.byref(ni), C.byref(no), C.byref(npt), C.byref(hm), C.byref(nr),
                                        None, counts))
        rots = (C.c_int32 * max(1, nr.value))()
        _check(lib().hy_conv_plan_query(self._p, None, None, None, None, None, rots, None))
        self.n_in, self.n_out, self.n_pt, self.has_mask = ni.value, no.value, npt.value, bool(hm.value)
        self.rots = [int(rots[i]) for i in range(nr.value)]
        self.counts = dict(zip(["Slide", "RaS", "RaS_g", "IR_g", "PMult"], [int(x) for x in counts]))
        eff = (C.c_uint32 * 5)()
        _check(lib().hy_conv_plan_eff_counts(self._p, eff))
        self.eff_counts = dict(zip(["Slide", "RaS", "RaS_g", "IR_g", "PMult"], [int(x) for x in eff]))

    def set_keyset(self, keyset):
        """Restrict the layer to a limited rotation-key set (hy_conv_plan_set_keyset): a KeySet or
        None (every key loaded).  self.rots becomes the loaded amounts the layer uses."""
        _check(lib().hy_conv_plan_set_keyset(self._p, keyset._k if keyset is not None else None))
        self._query()

    def __del__(self):
        if getattr(self, "_p", None) and getattr(self, "_lib", None) is not None:
            self._lib.hy_conv_plan_destroy(self._p)
            self._p = None

    def weight_slots(self, K, idx):
        K = np.ascontiguousarray(K, np.float64)
        out = np.zeros(self.n)
        _check(lib().hy_conv_weight_slots(self._p, K.ctypes.data_as(C.POINTER(C.c_double)), idx,
                                          out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def bias_slots(self, b, idx):
        b = np.ascontiguousarray(b, np.float64)
        out = np.zeros(self.n)
        _check(lib().hy_conv_bias_slots(self._p, b.ctypes.data_as(C.POINTER(C.c_double)), idx,
                                        out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def out_level(self, level):
        return level - 1 - int(self.has_mask)

    def encode_weights(self, K, level, bias=None, bias_scale=0):
        """weights (and mask) at `level`; with a bias plan, the bias plaintexts at the output level and scale
        bias_scale (the layer's ciphertext scale, an integer)."""
        words = int(lib().hy_conv_weight_words(self.ctx._c, self._p, level))
        pts = self.ctx.empty(max(words, 1))
        K = np.ascontiguousarray(K, np.float64)
        bp = None
        if bias is not None:
            b = np.ascontiguousarray(bias, np.float64)
            bp = b.ctypes.data_as(C.POINTER(C.c_double))
        _check(lib().hy_conv_encode_weights(self.ctx._c, self._p, K.ctypes.data_as(C.POINTER(C.c_double)), bp,
                                            int(bias_scale), level, _ptr(pts), self.ctx._stream()))
        return pts

    def scratch(self, level):
        return self.ctx.empty(int(lib().hy_conv_scratch_words(self.ctx._c, self._p, level)))

    def run(self, evks, cts, level, pts, scratch=None, out_begin=0, out_end=None, outs=None):
        """evks: dict rotation amount (mod n) -> key tensor, or a list in self.rots order."""
        if isinstance(evks, dict):
            evks = [evks[r] for r in self.rots]
        out_end = self.n_out if out_end is None else out_end
        lo = self.out_level(level)
        outs = [self.ctx.empty(*self.ctx.ct_shape(lo)) for _ in range(out_end - out_begin)] if outs is None else outs
        scratch = self.scratch(level) if scratch is None else scratch
        fn = lib().hy_caconv if self.algo == 0 else lib().hy_raconv
        _check(fn(self.ctx._c, self._p, _ptr_array(evks), _ptr_array(cts), level, _ptr(pts), _ptr(scratch),
                  out_begin, out_end, _ptr_array(outs), self.ctx._stream()))
        return outs

    # ---- CAConv Slide sharding (include/hyphen.h hy_caconv_slide / hy_caconv_slid)
    def slide(self, evks, cts, level, in_begin=0, in_end=None, out=None):
        """Slide_f of inputs [in_begin, in_end) -> [(in_end - in_begin) * f^2][2][l+1][N] (hy_caconv_slide)"""
        if isinstance(evks, dict):
            evks = [evks[r] for r in self.rots]
        in_end = self.n_in if in_end is None else in_end
        f2 = self.f * self.f
        out = self.ctx.empty((in_end - in_begin) * f2, *self.ctx.ct_shape(level)) if out is None else out
        if in_end > in_begin:
            _check(lib().hy_caconv_slide(self.ctx._c, self._p, _ptr_array(evks), _ptr_array(cts), level, in_begin,
                                         in_end, _ptr(out), self.ctx._stream()))
        return out

    def run_slid(self, evks, slid, level, pts, scratch=None, out_begin=0, out_end=None, outs=None):
        """the layer from a complete slid buffer (hy_caconv_slid)"""
        if isinstance(evks, dict):
            evks = [evks[r] for r in self.rots]
        out_end = self.n_out if out_end is None else out_end
        lo = self.out_level(level)
        outs = [self.ctx.empty(*self.ctx.ct_shape(lo)) for _ in range(out_end - out_begin)] if outs is None else outs
        scratch = self.scratch(level) if scratch is None else scratch
        _check(lib().hy_caconv_slid(self.ctx._c, self._p, _ptr_array(evks), _ptr(slid), level, _ptr(pts),
                                    _ptr(scratch), out_begin, out_end, _ptr_array(outs), self.ctx._stream()))
        return outs

    # ---- RAConv tap sharding (include/hyphen.h hy_raconv_partial / hy_raconv_finish)
    def partial_state(self, level):
        """An int64 device buffer for the lazy-sum state of one output (summable across ranks)."""
        return self.ctx.zeros(int(lib().hy_raconv_partial_words(self.ctx._c, level)))

    def raconv_partial(self, evks, cts, level, pts, out_index, tap_begin, tap_end, state, scratch=None):
        if isinstance(evks, dict):
            evks = [evks[r] for r in self.rots]
        scratch = self.scratch(level) if scratch is None else scratch
        _check(lib().hy_raconv_partial(self.ctx._c, self._p, _ptr_array(evks), _ptr_array(cts), level, _ptr(pts),
                                       _ptr(scratch), out_index, tap_begin, tap_end, _ptr(state),
                                       self.ctx._stream()))
        return state

    def raconv_finish(self, evks, level, pts, state, out_index, out=None, scratch=None):
        if isinstance(evks, dict):
            evks = [evks[r] for r in self.rots]
        out = self.ctx.empty(*self.ctx.ct_shape(self.out_level(level))) if out is None else out
        scratch = self.scratch(level) if scratch is None else scratch
        _check(lib().hy_raconv_finish(self.ctx._c, self._p, _ptr_array(evks), level, _ptr(pts), _ptr(state),
                                      _ptr(scratch), out_index, _ptr(out), self.ctx._stream()))
        return out


class ConvBlock:
    """The conv half of a ResNet basic block as HyPHEN fuses it (Alg. 3): CAConv, the AESPA activation
    with its coefficients fused into the neighbouring layers -- x^2, MulCt + relinearization +
    rescale, one level -- then RAConv.  Every step is a C-ABI call (hy_caconv, hy_mulct_batch, hy_rescale,
    hy_raconv); the paper interleaves the loops only to bound the live ciphertexts, which 180 GB of HBM does
    not need, and modular sums do not depend on that order (identical limbs)."""

    def __init__(self, ctx, ca: "ConvPlan", ra: "ConvPlan"):
        assert ca.algo == ConvPlan.CA and ra.algo == ConvPlan.RA
        assert ca.n_out == ra.n_in, "CAConv outputs must be the RAConv inputs"
        self.ctx, self.ca, self.ra = ctx, ca, ra

    def levels(self, level):
        """(CAConv output, RAConv input, block output) levels for a block input at `level`."""
        mid = self.ca.out_level(level)
        return mid, mid - 1, self.ra.out_level(mid - 1)

    def run(self, ca_evks, ra_evks, rlk, cts, level, ca_pts, ra_pts, ca_scratch=None, ra_scratch=None):
        mid, ra_level, _ = self.levels(level)
        x = self.ca.run(ca_evks, cts, level, ca_pts, ca_scratch)
        x = self.ctx.square_batch(rlk, x, mid, outs=x)
        x = [self.ctx.rescale(c, mid) for c in x]
        return self.ra.run(ra_evks, x, ra_level, ra_pts, ra_scratch)
