"""CPU oracle for HyPHEN's homomorphic-convolution hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2302_02407_b200``) never imports it and shares no code with it.

``ckks_oracle.c`` (plain C, ``__int128 %`` arithmetic, textbook NTT) holds the
RNS-CKKS operations; this module wraps it with ctypes and adds the pieces that
are easier to read in Python: decode (big-int CRT + numpy FFT) and the HyPHEN
layer code in ``oracle.hyphen``.  See the C file header for citations.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ckks_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

DOM_SK, DOM_EVK_A, DOM_EVK_E, DOM_ENC_A, DOM_ENC_E = 1, 2, 3, 4, 5


def build(force: bool = False) -> str:
    """Compile the C oracle (gcc, -O2, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", _LIB, _SRC, "-lquadmath"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        P = C.c_void_p
        u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
        i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
        i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
        i8p = np.ctypeslib.ndpointer(np.int8, flags="C_CONTIGUOUS")
        u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
        f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
        ip = C.POINTER(C.c_int)
        sig = {
            "orc_ctx_new": (P, [C.c_int, C.c_int, ip, C.c_int, ip, C.c_int]),
            "orc_ctx_free": (None, [P]),
            "orc_ctx_moduli": (None, [P, u64p]),
            "orc_ctx_psi": (None, [P, u64p]),
            "orc_ctx_alpha": (C.c_int, [P]),
            "orc_n_digits": (C.c_int, [P, C.c_int]),
            "orc_is_prime": (C.c_int, [C.c_uint64]),
            "orc_philox4x32_10": (None, [u32p, u32p, u32p]),
            "orc_ntt": (None, [P, C.c_int, u64p]),
            "orc_intt": (None, [P, C.c_int, u64p]),
            "orc_automorph_coeff": (None, [P, C.c_int, C.c_uint64, u64p, u64p]),
            "orc_galois_elt": (C.c_uint64, [P, C.c_int64]),
            "orc_sample_secret": (None, [P, C.c_uint64, C.c_int, i8p]),
            "orc_sample_cbd": (None, [C.c_uint64, C.c_uint32, C.c_uint64, C.c_int, i32p]),
            "orc_keygen_rot": (None, [P, C.c_uint64, C.c_int, C.c_uint64, C.c_uint64, u64p]),
            "orc_encrypt": (None, [P, C.c_uint64, C.c_int, C.c_uint64, C.c_uint64, u64p, C.c_int, u64p]),
            "orc_decrypt": (None, [P, C.c_uint64, C.c_int, u64p, C.c_int, u64p]),
            "orc_encode_coeffs": (C.c_int, [P, f64p, P, C.c_uint64, i64p]),
            "orc_coeffs_to_pt": (None, [P, i64p, C.c_int, u64p]),
            "orc_modup_coeff": (None, [P, C.c_int, u64p, u64p]),
            "orc_ks_inner_product": (None, [P, C.c_int, u64p, u64p, u64p]),
            "orc_moddown": (None, [P, C.c_int, u64p, u64p]),
            "orc_hrot": (None, [P, C.c_int, u64p, C.c_uint64, u64p, u64p]),
            "orc_hrot_hoisted": (None, [P, C.c_int, P, u64p, C.c_int, u64p, P]),
            "orc_hrot_sum": (None, [P, C.c_int, P, u64p, C.c_int, P, u64p]),
            "orc_pmult": (None, [P, C.c_int, u64p, u64p, u64p]),
            "orc_add": (None, [P, C.c_int, C.c_int, u64p, u64p, u64p]),
            "orc_rescale": (None, [P, C.c_int, u64p, u64p]),
            "orc_keygen_relin": (None, [P, C.c_uint64, C.c_int, C.c_uint64, u64p]),
            "orc_mulct": (None, [P, C.c_int, u64p, u64p, u64p, u64p]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _ptr_array(arrs):
    a = (C.c_void_p * len(arrs))()
    for i, x in enumerate(arrs):
        assert x.dtype == np.uint64 and x.flags["C_CONTIGUOUS"]
        a[i] = x.ctypes.data
    return a


def philox4x32_10(key, ctr):
    out = np.zeros(4, np.uint32)
    lib().orc_philox4x32_10(np.asarray(key, np.uint32), np.asarray(ctr, np.uint32), out)
    return out


def is_prime(n: int) -> bool:
    return bool(lib().orc_is_prime(n))


@dataclass
class Ct:
    """ciphertext: data [2][level+1][N] uint64, NTT domain; scale tracked exactly as a float."""
    data: np.ndarray
    level: int
    scale: float


@dataclass
class Pt:
    data: np.ndarray  # [level+1][N] uint64, NTT domain
    level: int
    scale: float


class Oracle:
    """RNS-CKKS oracle context for one parameter set (see synth.PARAMS)."""

    def __init__(self, log_n, q_bits, p_bits, dnum, h=192, log_scale=40, **_):
        self.log_n, self.N, self.n = log_n, 1 << log_n, 1 << (log_n - 1)
        self.nq, self.np_, self.dnum, self.h = len(q_bits), len(p_bits), dnum, h
        self.log_scale = log_scale
        qb = (C.c_int * len(q_bits))(*q_bits)
        pb = (C.c_int * len(p_bits))(*p_bits)
        self._c = lib().orc_ctx_new(log_n, len(q_bits), qb, len(p_bits), pb, dnum)
        if not self._c:
            raise ValueError("oracle context creation failed")
        self.moduli = np.zeros(self.nq + self.np_, np.uint64)
        lib().orc_ctx_moduli(self._c, self.moduli)
        self.psi = np.zeros(self.nq + self.np_, np.uint64)
        lib().orc_ctx_psi(self._c, self.psi)
        self.alpha = lib().orc_ctx_alpha(self._c)
        self.q = [int(x) for x in self.moduli[: self.nq]]
        self.p = [int(x) for x in self.moduli[self.nq:]]

    def __del__(self):
        if getattr(self, "_c", None):
            lib().orc_ctx_free(self._c)
            self._c = None

    # -- basic transforms ------------------------------------------------
    def ntt(self, a, chain_idx):
        a = np.ascontiguousarray(a, np.uint64).copy()
        lib().orc_ntt(self._c, chain_idx, a)
        return a

    def intt(self, a, chain_idx):
        a = np.ascontiguousarray(a, np.uint64).copy()
        lib().orc_intt(self._c, chain_idx, a)
        return a

    def automorph_coeff(self, a, chain_idx, k):
        out = np.zeros(self.N, np.uint64)
        lib().orc_automorph_coeff(self._c, chain_idx, k, np.ascontiguousarray(a, np.uint64), out)
        return out

    def galois_elt(self, r: int) -> int:
        return int(lib().orc_galois_elt(self._c, int(r)))

    def n_digits(self, level: int) -> int:
        return int(lib().orc_n_digits(self._c, level))

    def ext_chain(self, level):
        return list(range(level + 1)) + [self.nq + k for k in range(self.np_)]

    def to_ntt(self, coeffs_limbs, chain):
        return np.stack([self.ntt(coeffs_limbs[u], chain[u]) for u in range(len(chain))])

    def to_coeff(self, ntt_limbs, chain):
        return np.stack([self.intt(ntt_limbs[u], chain[u]) for u in range(len(chain))])

    # -- sampling / keys -------------------------------------------------
    def secret(self, sk_seed):
        s = np.zeros(self.N, np.int8)
        lib().orc_sample_secret(self._c, sk_seed, self.h, s)
        return s

    def cbd(self, seed, dom, obj):
        e = np.zeros(self.N, np.int32)
        lib().orc_sample_cbd(seed, dom, obj, self.N, e)
        return e

    def keygen_rot(self, sk_seed, ek_seed, r: int):
        """rotation key for a left rotation by r; [dnum][2][nq+np][N]."""
        return self.keygen_galois(sk_seed, ek_seed, self.galois_elt(r))

    def keygen_galois(self, sk_seed, ek_seed, k: int):
        evk = np.zeros((self.dnum, 2, self.nq + self.np_, self.N), np.uint64)
        lib().orc_keygen_rot(self._c, sk_seed, self.h, ek_seed, k, evk)
        return evk

    def keygen_relin(self, sk_seed, ek_seed):
        """relinearization key s^2 -> s (DESIGN R-RELIN); [dnum][2][nq+np][N]."""
        evk = np.zeros((self.dnum, 2, self.nq + self.np_, self.N), np.uint64)
        lib().orc_keygen_relin(self._c, sk_seed, self.h, ek_seed, evk)
        return evk

    # -- encode / encrypt ------------------------------------------------
    def encode_coeffs(self, z, scale: int):
        z = np.asarray(z)
        re = np.ascontiguousarray(np.real(z), np.float64)
        im = np.ascontiguousarray(np.imag(z), np.float64) if np.iscomplexobj(z) else None
        if len(re) < self.n:
            re = np.concatenate([re, np.zeros(self.n - len(re))])
            if im is not None:
                im = np.concatenate([im, np.zeros(self.n - len(im))])
        out = np.zeros(self.N, np.int64)
        rc = lib().orc_encode_coeffs(self._c, re, im.ctypes.data if im is not None else None, int(scale), out)
        if rc != 0:
            raise OverflowError("encoded coefficient exceeds 2^62")
        return out

    def coeffs_to_pt(self, coeffs, level):
        pt = np.zeros((level + 1, self.N), np.uint64)
        lib().orc_coeffs_to_pt(self._c, np.ascontiguousarray(coeffs, np.int64), level, pt)
        return pt

    def encode(self, z, scale: int, level: int) -> Pt:
        return Pt(self.coeffs_to_pt(self.encode_coeffs(z, scale), level), level, float(scale))

    def encrypt(self, sk_seed, enc_seed, ct_id, pt: Pt) -> Ct:
        ct = np.zeros((2, pt.level + 1, self.N), np.uint64)
        lib().orc_encrypt(self._c, sk_seed, self.h, enc_seed, ct_id, np.ascontiguousarray(pt.data), pt.level, ct)
        return Ct(ct, pt.level, pt.scale)

    def decrypt(self, sk_seed, ct: Ct) -> Pt:
        m = np.zeros((ct.level + 1, self.N), np.uint64)
        lib().orc_decrypt(self._c, sk_seed, self.h, np.ascontiguousarray(ct.data), ct.level, m)
        return Pt(m, ct.level, ct.scale)

    # -- decode (Python big-int CRT + float64 FFT; tolerance-checked) ------
    def crt_coeffs(self, pt_data, level):
        """NTT-domain limbs on q_0..q_level -> centred integer coefficients (Python ints)."""
        coeff = [self.intt(pt_data[i], i) for i in range(level + 1)]
        Q = 1
        for i in range(level + 1):
            Q *= self.q[i]
        out = [0] * self.N
        terms = []
        for i in range(level + 1):
            Qi = Q // self.q[i]
            terms.append((Qi, pow(Qi, -1, self.q[i])))
        for x in range(self.N):
            v = 0
            for i in range(level + 1):
                Qi, inv = terms[i]
                v += (int(coeff[i][x]) * inv % self.q[i]) * Qi
            v %= Q
            if v > Q // 2:
                v -= Q
            out[x] = v
        return out

    def decode(self, pt: Pt):
        """complex slot values z_j = m(zeta^{5^j}) / scale, zeta = exp(i pi / N)."""
        m = np.array([float(v) for v in self.crt_coeffs(pt.data, pt.level)], dtype=np.float64)
        return self.eval_slots(m) / pt.scale

    def eval_slots(self, m):
        """evaluate real coefficient vector m at zeta^{5^j}, j < n (canonical embedding)."""
        twoN = 2 * self.N
        M = np.fft.ifft(np.concatenate([m, np.zeros(self.N)])) * twoN  # sum_k m_k exp(+2 pi i e k / 2N)
        idx = np.array([pow(5, j, twoN) for j in range(self.n)])
        return M[idx]

    # -- key switching ---------------------------------------------------
    def modup_coeff(self, level, d_coeff):
        E = level + 1 + self.np_
        out = np.zeros((self.n_digits(level), E, self.N), np.uint64)
        lib().orc_modup_coeff(self._c, level, np.ascontiguousarray(d_coeff, np.uint64), out)
        return out

    def ks_inner_product(self, level, ext, evk):
        E = level + 1 + self.np_
        u = np.zeros((2, E, self.N), np.uint64)
        lib().orc_ks_inner_product(self._c, level, np.ascontiguousarray(ext), np.ascontiguousarray(evk), u)
        return u

    def moddown(self, level, u_poly):
        out = np.zeros((level + 1, self.N), np.uint64)
        lib().orc_moddown(self._c, level, np.ascontiguousarray(u_poly), out)
        return out

    def hrot(self, ct: Ct, evk, r: int) -> Ct:
        out = np.zeros_like(ct.data)
        lib().orc_hrot(self._c, ct.level, np.ascontiguousarray(evk), self.galois_elt(r), np.ascontiguousarray(ct.data), out)
        return Ct(out, ct.level, ct.scale)

    def hrot_galois(self, ct: Ct, evk, k: int) -> Ct:
        """key switch by any Galois element k (k = 2N - 1: conjugation), the plain variant"""
        out = np.zeros_like(ct.data)
        lib().orc_hrot(self._c, ct.level, np.ascontiguousarray(evk), int(k), np.ascontiguousarray(ct.data), out)
        return Ct(out, ct.level, ct.scale)

    def hrot_hoisted(self, ct: Ct, evks, rs):
        outs = [np.zeros_like(ct.data) for _ in rs]
        ks = np.array([self.galois_elt(r) for r in rs], np.uint64)
        evk_list = [np.ascontiguousarray(e) for e in evks]
        lib().orc_hrot_hoisted(self._c, ct.level, _ptr_array(evk_list), ks, len(rs),
                               np.ascontiguousarray(ct.data), _ptr_array(outs))
        return [Ct(o, ct.level, ct.scale) for o in outs]

    def hrot_sum(self, cts, evks, rs) -> Ct:
        level = cts[0].level
        assert all(c.level == level for c in cts)
        out = np.zeros_like(cts[0].data)
        ks = np.array([self.galois_elt(r) for r in rs], np.uint64)
        evk_list = [np.ascontiguousarray(e) if e is not None else np.zeros(1, np.uint64) for e in evks]
        data = [np.ascontiguousarray(c.data) for c in cts]
        lib().orc_hrot_sum(self._c, level, _ptr_array(evk_list), ks, len(rs), _ptr_array(data), out)
        return Ct(out, level, cts[0].scale)

    # -- MulPt / AddCt / Rescale -----------------------------------------
    def pmult(self, ct: Ct, pt: Pt) -> Ct:
        assert ct.level == pt.level
        out = np.zeros_like(ct.data)
        lib().orc_pmult(self._c, ct.level, np.ascontiguousarray(ct.data), np.ascontiguousarray(pt.data), out)
        return Ct(out, ct.level, ct.scale * pt.scale)

    def add(self, a: Ct, b: Ct) -> Ct:
        assert a.level == b.level
        out = np.zeros_like(a.data)
        lib().orc_add(self._c, a.level, 2, np.ascontiguousarray(a.data), np.ascontiguousarray(b.data), out)
        return Ct(out, a.level, a.scale)

    def add_pt(self, a: Ct, pt: Pt) -> Ct:
        """AddPt: plaintext added to c0."""
        out = a.data.copy()
        o0 = np.zeros_like(a.data[0])
        lib().orc_add(self._c, a.level, 1, np.ascontiguousarray(a.data[0]), np.ascontiguousarray(pt.data), o0)
        out[0] = o0
        return Ct(out, a.level, a.scale)

    def rescale(self, ct: Ct) -> Ct:
        assert ct.level >= 1
        out = np.zeros((2, ct.level, self.N), np.uint64)
        lib().orc_rescale(self._c, ct.level, np.ascontiguousarray(ct.data), out)
        return Ct(out, ct.level - 1, ct.scale / self.q[ct.level])

    def mulct(self, a: Ct, b: Ct, rlk) -> Ct:
        """MulCt + relinearization, no rescale; scale a.scale * b.scale."""
        assert a.level == b.level
        out = np.zeros_like(a.data)
        lib().orc_mulct(self._c, a.level, np.ascontiguousarray(a.data), np.ascontiguousarray(b.data),
                        np.ascontiguousarray(rlk), out)
        return Ct(out, a.level, a.scale * b.scale)

    def square(self, a: Ct, rlk) -> Ct:
        """AESPA activation after its coefficients are fused into the neighbouring layers: x^2,
        MulCt(a, a) + relinearization + rescale."""
        return self.rescale(self.mulct(a, a, rlk))

    def level_down(self, ct: Ct, level: int) -> Ct:
        assert level <= ct.level
        return Ct(np.ascontiguousarray(ct.data[:, : level + 1]), level, ct.scale)
