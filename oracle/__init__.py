"""CPU oracle for hybrid key switching -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2507_04775_b200``) never imports it and shares no code with it.

The arithmetic lives in ``oracle/oracle.c`` (plain C, ``%`` on ``unsigned __int128``);
this module only marshals numpy arrays into it and adds the harness-side client
operations (key generation, encryption of a test message, decryption with big-int
CRT reconstruction) used by the noise-bound pins.

Parity status: every function exported here is pinned
by a ``-m "not gpu"`` test in ``tests/test_oracle_*.py`` against something other than
itself (schoolbook products, closed forms, CRT/big-int invariants, decryption bound).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.c")

_u64p = ctypes.POINTER(ctypes.c_uint64)
_u32p = ctypes.POINTER(ctypes.c_uint32)
_i64p = ctypes.POINTER(ctypes.c_int64)
_vp = ctypes.c_void_p


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc -O2 -fopenmp (plain C; building the checker is not using it)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", tmp, _SRC])
        os.replace(tmp, _SO)
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        L.or_ctx_new.restype = _vp
        L.or_ctx_new.argtypes = [ctypes.c_uint32, _u64p, ctypes.c_uint32, _u64p, ctypes.c_uint32, ctypes.c_uint32]
        L.or_ctx_free.argtypes = [_vp]
        L.or_ctx_psi.restype = ctypes.c_uint64
        L.or_ctx_psi.argtypes = [_vp, ctypes.c_uint32]
        L.or_min_psi.restype = ctypes.c_uint64
        L.or_min_psi.argtypes = [ctypes.c_uint64, ctypes.c_uint32]
        L.or_is_prime.restype = ctypes.c_int
        L.or_is_prime.argtypes = [ctypes.c_uint64]
        L.or_beta.restype = ctypes.c_uint32
        L.or_beta.argtypes = [_vp, ctypes.c_uint32]
        for name in ("or_ntt", "or_intt"):
            getattr(L, name).argtypes = [_vp, _u64p, _u32p, ctypes.c_uint32]
        L.or_ntt_def.argtypes = [_vp, _u64p, ctypes.c_uint32, _u32p, ctypes.c_uint32, _u64p]
        for name in ("or_add", "or_sub", "or_mul"):
            getattr(L, name).argtypes = [_vp, _u64p, _u64p, _u32p, ctypes.c_uint32, _u64p]
        L.or_lift.argtypes = [_vp, _i64p, _u32p, ctypes.c_uint32, _u64p]
        L.or_automorph_coeff.argtypes = [_vp, _u64p, _u32p, ctypes.c_uint32, ctypes.c_uint64, _u64p]
        L.or_automorph.argtypes = [_vp, _u64p, ctypes.c_uint32, ctypes.c_uint64, _u64p]
        L.or_bconv.argtypes = [_vp, _u64p, _u32p, ctypes.c_uint32, _u32p, ctypes.c_uint32, _u64p]
        L.or_modup.argtypes = [_vp, _u64p, ctypes.c_uint32, _u64p]
        L.or_kip.argtypes = [_vp, _u64p, _u64p, ctypes.c_uint32, ctypes.c_uint64, _u64p]
        L.or_moddown.argtypes = [_vp, _u64p, ctypes.c_uint32, _u64p]
        L.or_keyswitch.argtypes = [_vp, _u64p, _u64p, ctypes.c_uint32, _u64p, _u64p, _u64p]
        L.or_rotate.argtypes = [_vp, _u64p, _u64p, ctypes.c_uint32, ctypes.c_uint64, _u64p, _u64p, _u64p]
        L.or_rotate_hoisted.argtypes = [_vp, _u64p, _u64p, ctypes.c_uint32, ctypes.c_uint32, _u64p,
                                        ctypes.POINTER(_u64p), ctypes.POINTER(_u64p), ctypes.POINTER(_u64p)]
        L.or_tensor.argtypes = [_vp, _u64p, _u64p, _u64p, _u64p, ctypes.c_uint32, _u64p, _u64p, _u64p]
        L.or_hmult.argtypes = [_vp, _u64p, _u64p, _u64p, _u64p, ctypes.c_uint32, _u64p, _u64p, _u64p]
        L.or_rescale.argtypes = [_vp, _u64p, ctypes.c_uint32, _u64p]
        _pp = ctypes.POINTER(_u64p)
        L.or_pt_wsum.argtypes = [_vp, ctypes.c_uint32, _pp, _pp, _pp, ctypes.c_uint32, _u64p, _u64p]
        L.or_lintrans.argtypes = [_vp, _u64p, _u64p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, _u64p, _pp,
                                  _u64p, _pp, _pp, _u64p, _u64p]
        L.or_keygen_ks.argtypes = [_vp, _u64p, _u64p, _u64p, _i64p, _u64p]
        L.or_decrypt.argtypes = [_vp, _u64p, _u64p, ctypes.c_uint32, _u64p, _u64p]
        _lib = L
    return _lib


def _p64(a: np.ndarray):
    assert a.dtype == np.uint64 and a.flags.c_contiguous
    return a.ctypes.data_as(_u64p)


def _pi64(a: np.ndarray):
    assert a.dtype == np.int64 and a.flags.c_contiguous
    return a.ctypes.data_as(_i64p)


def _p32(seq) -> tuple:
    arr = np.ascontiguousarray(np.asarray(seq, dtype=np.uint32))
    return arr, arr.ctypes.data_as(_u32p)


def set_num_threads(n: int) -> int:
    """OpenMP threads of the oracle's parallel loops (independent limbs / coefficients); returns the previous
    count.  Timing only (bench.py cpu_baseline single-thread leg): results do not depend on it."""
    L = lib()
    L.omp_get_max_threads.restype = ctypes.c_int
    prev = int(L.omp_get_max_threads())
    L.omp_set_num_threads(ctypes.c_int(int(n)))
    return prev


def is_prime(n: int) -> bool:
    return bool(lib().or_is_prime(n))


def min_psi(p: int, n: int) -> int:
    return int(lib().or_min_psi(p, n))


class Ctx:
    """Oracle context for (N, q chain, special primes P, dnum)."""

    def __init__(self, log_n: int, q, p, dnum: int):
        self.log_n, self.n = log_n, 1 << log_n
        self.q, self.p, self.dnum = tuple(int(x) for x in q), tuple(int(x) for x in p), dnum
        self.nq, self.np = len(self.q), len(self.p)
        self.primes = self.q + self.p
        self.alpha = -(-self.nq // dnum)
        qa = np.array(self.q, dtype=np.uint64)
        pa = np.array(self.p, dtype=np.uint64)
        self._h = lib().or_ctx_new(log_n, _p64(qa), self.nq, _p64(pa), self.np, dnum)
        if not self._h:
            raise ValueError("oracle: invalid parameters")

    @classmethod
    def from_config(cls, cfg):
        return cls(cfg.log_n, cfg.q, cfg.p, cfg.dnum)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.or_ctx_free(h)
            self._h = None

    # ---- structure
    def psi(self, idx: int) -> int:
        return int(lib().or_ctx_psi(self._h, idx))

    def beta(self, level: int) -> int:
        return int(lib().or_beta(self._h, level))

    def digits(self, level: int):
        return [(j * self.alpha, min((j + 1) * self.alpha, level + 1)) for j in range(self.beta(level))]

    def ext_primes(self, level: int):
        return list(range(level + 1)) + [self.nq + k for k in range(self.np)]

    # ---- transforms
    def ntt(self, x: np.ndarray, idx) -> np.ndarray:
        y = np.ascontiguousarray(x, dtype=np.uint64).copy()
        ia, ip = _p32(idx)
        assert y.shape == (len(ia), self.n)
        lib().or_ntt(self._h, _p64(y), ip, len(ia))
        return y

    def intt(self, x: np.ndarray, idx) -> np.ndarray:
        y = np.ascontiguousarray(x, dtype=np.uint64).copy()
        ia, ip = _p32(idx)
        assert y.shape == (len(ia), self.n)
        lib().or_intt(self._h, _p64(y), ip, len(ia))
        return y

    def ntt_def(self, a: np.ndarray, pidx: int, js) -> np.ndarray:
        a = np.ascontiguousarray(a, dtype=np.uint64)
        ja, jp = _p32(js)
        out = np.zeros(len(ja), dtype=np.uint64)
        lib().or_ntt_def(self._h, _p64(a), pidx, jp, len(ja), _p64(out))
        return out

    # ---- elementwise
    def _ew(self, fn, a, b, idx):
        a = np.ascontiguousarray(a, dtype=np.uint64)
        b = np.ascontiguousarray(b, dtype=np.uint64)
        out = np.empty_like(a)
        ia, ip = _p32(idx)
        fn(self._h, _p64(a), _p64(b), ip, len(ia), _p64(out))
        return out

    def add(self, a, b, idx):
        return self._ew(lib().or_add, a, b, idx)

    def sub(self, a, b, idx):
        return self._ew(lib().or_sub, a, b, idx)

    def mul(self, a, b, idx):
        return self._ew(lib().or_mul, a, b, idx)

    def lift(self, coef: np.ndarray, idx) -> np.ndarray:
        coef = np.ascontiguousarray(coef, dtype=np.int64)
        ia, ip = _p32(idx)
        out = np.empty((len(ia), self.n), dtype=np.uint64)
        lib().or_lift(self._h, _pi64(coef), ip, len(ia), _p64(out))
        return out

    def automorph_coeff(self, x, idx, galois: int):
        x = np.ascontiguousarray(x, dtype=np.uint64)
        ia, ip = _p32(idx)
        out = np.empty_like(x)
        lib().or_automorph_coeff(self._h, _p64(x), ip, len(ia), galois, _p64(out))
        return out

    def automorph(self, x, galois: int):
        x = np.ascontiguousarray(x, dtype=np.uint64)
        out = np.empty_like(x)
        lib().or_automorph(self._h, _p64(x), x.shape[0], galois, _p64(out))
        return out

    # ---- key-switching steps
    def bconv(self, x, src, dst):
        x = np.ascontiguousarray(x, dtype=np.uint64)
        sa, sp = _p32(src)
        da, dp = _p32(dst)
        out = np.empty((len(da), self.n), dtype=np.uint64)
        lib().or_bconv(self._h, _p64(x), sp, len(sa), dp, len(da), _p64(out))
        return out

    def modup(self, d, level: int):
        d = np.ascontiguousarray(d, dtype=np.uint64)
        assert d.shape == (level + 1, self.n)
        ext = np.zeros((self.beta(level), level + 1 + self.np, self.n), dtype=np.uint64)
        lib().or_modup(self._h, _p64(d), level, _p64(ext))
        return ext

    def kip(self, ext, evk, level: int, galois: int = 1):
        ext = np.ascontiguousarray(ext, dtype=np.uint64)
        evk = np.ascontiguousarray(evk, dtype=np.uint64)
        acc = np.zeros((2, level + 1 + self.np, self.n), dtype=np.uint64)
        lib().or_kip(self._h, _p64(ext), _p64(evk), level, galois, _p64(acc))
        return acc

    def moddown(self, acc, level: int):
        acc = np.ascontiguousarray(acc, dtype=np.uint64)
        assert acc.shape == (level + 1 + self.np, self.n)
        out = np.empty((level + 1, self.n), dtype=np.uint64)
        lib().or_moddown(self._h, _p64(acc), level, _p64(out))
        return out

    def keyswitch(self, c0, c1, evk, level: int):
        c0 = np.ascontiguousarray(c0, dtype=np.uint64)
        c1 = np.ascontiguousarray(c1, dtype=np.uint64)
        evk = np.ascontiguousarray(evk, dtype=np.uint64)
        out0 = np.empty_like(c0)
        out1 = np.empty_like(c1)
        lib().or_keyswitch(self._h, _p64(c0), _p64(c1), level, _p64(evk), _p64(out0), _p64(out1))
        return out0, out1

    def rotate(self, c0, c1, evk, level: int, galois: int):
        c0 = np.ascontiguousarray(c0, dtype=np.uint64)
        c1 = np.ascontiguousarray(c1, dtype=np.uint64)
        evk = np.ascontiguousarray(evk, dtype=np.uint64)
        out0, out1 = np.empty_like(c0), np.empty_like(c1)
        lib().or_rotate(self._h, _p64(c0), _p64(c1), level, galois, _p64(evk), _p64(out0), _p64(out1))
        return out0, out1

    def rotate_hoisted(self, c0, c1, evks, level: int, galois):
        c0 = np.ascontiguousarray(c0, dtype=np.uint64)
        c1 = np.ascontiguousarray(c1, dtype=np.uint64)
        evks = [np.ascontiguousarray(e, dtype=np.uint64) for e in evks]
        nrot = len(evks)
        outs0 = [np.empty_like(c0) for _ in range(nrot)]
        outs1 = [np.empty_like(c1) for _ in range(nrot)]
        g = np.array(galois, dtype=np.uint64)
        ek = (_u64p * nrot)(*[_p64(e) for e in evks])
        o0 = (_u64p * nrot)(*[_p64(o) for o in outs0])
        o1 = (_u64p * nrot)(*[_p64(o) for o in outs1])
        lib().or_rotate_hoisted(self._h, _p64(c0), _p64(c1), level, nrot, _p64(g), ek, o0, o1)
        return outs0, outs1

    # ---- HMult front-end and Rescale (oracle.c: or_tensor, or_hmult, or_rescale)
    def tensor(self, a0, a1, b0, b1, level: int):
        a0, a1, b0, b1 = (np.ascontiguousarray(v, dtype=np.uint64) for v in (a0, a1, b0, b1))
        d0, d1, d2 = np.empty_like(a0), np.empty_like(a0), np.empty_like(a0)
        lib().or_tensor(self._h, _p64(a0), _p64(a1), _p64(b0), _p64(b1), level, _p64(d0), _p64(d1), _p64(d2))
        return d0, d1, d2

    def hmult(self, a0, a1, b0, b1, evk, level: int):
        a0, a1, b0, b1 = (np.ascontiguousarray(v, dtype=np.uint64) for v in (a0, a1, b0, b1))
        evk = np.ascontiguousarray(evk, dtype=np.uint64)
        out0, out1 = np.empty_like(a0), np.empty_like(a0)
        lib().or_hmult(self._h, _p64(a0), _p64(a1), _p64(b0), _p64(b1), level, _p64(evk), _p64(out0), _p64(out1))
        return out0, out1

    def rescale(self, x, level: int):
        """One polynomial [l+1][N] EVAL at level l -> [l][N] EVAL at level l-1."""
        assert level >= 1
        x = np.ascontiguousarray(x, dtype=np.uint64)
        assert x.shape == (level + 1, self.n)
        out = np.empty((level, self.n), dtype=np.uint64)
        lib().or_rescale(self._h, _p64(x), level, _p64(out))
        return out

    # ---- BSGS linear transform (oracle.c: or_pt_wsum, or_lintrans)
    def pt_wsum(self, w, x0, x1, level: int):
        w, x0, x1 = ([np.ascontiguousarray(v, dtype=np.uint64) for v in arr] for arr in (w, x0, x1))
        n = len(w)
        arr = lambda vs: (_u64p * n)(*[_p64(v) for v in vs])
        out0, out1 = np.empty_like(x0[0]), np.empty_like(x0[0])
        lib().or_pt_wsum(self._h, n, arr(w), arr(x0), arr(x1), level, _p64(out0), _p64(out1))
        return out0, out1

    def lintrans(self, c0, c1, level: int, n1: int, n2: int, baby_galois, baby_keys, giant_galois, giant_keys, pts):
        """pts: n2*n1 diagonals [l+1][N] (index i*n1 + j); baby/giant lists have n1-1 / n2-1 entries."""
        c0 = np.ascontiguousarray(c0, dtype=np.uint64)
        c1 = np.ascontiguousarray(c1, dtype=np.uint64)
        keep = [np.ascontiguousarray(v, dtype=np.uint64) for v in list(baby_keys) + list(giant_keys) + list(pts)]
        nb, ng = len(baby_keys), len(giant_keys)
        assert nb == n1 - 1 and ng == n2 - 1 and len(pts) == n1 * n2
        arr = lambda vs: (_u64p * max(1, len(vs)))(*[_p64(v) for v in vs])
        bg = np.array(list(baby_galois) + [1], dtype=np.uint64)
        gg = np.array(list(giant_galois) + [1], dtype=np.uint64)
        out0, out1 = np.empty_like(c0), np.empty_like(c0)
        lib().or_lintrans(self._h, _p64(c0), _p64(c1), level, n1, n2, _p64(bg), arr(keep[:nb]), _p64(gg),
                          arr(keep[nb:nb + ng]), arr(keep[nb + ng:]), _p64(out0), _p64(out1))
        return out0, out1

    # ---- client side (harness only)
    def secret_eval(self, s_coef: np.ndarray) -> np.ndarray:
        """Ternary secret lifted to all L+1+K limbs, EVAL form."""
        idx = list(range(self.nq + self.np))
        return self.ntt(self.lift(s_coef, idx), idx)

    def keygen_ks(self, s_eval, s_old_eval, a, e):
        """evk [dnum][2][L+1+K][N]; a, e are drawn by hks_synth and passed in."""
        nk = self.nq + self.np
        a = np.ascontiguousarray(a, dtype=np.uint64)
        e = np.ascontiguousarray(e, dtype=np.int64)
        assert a.shape == (self.dnum, nk, self.n) and e.shape == (self.dnum, self.n)
        evk = np.empty((self.dnum, 2, nk, self.n), dtype=np.uint64)
        lib().or_keygen_ks(self._h, _p64(np.ascontiguousarray(s_eval)), _p64(np.ascontiguousarray(s_old_eval)),
                           _p64(a), _pi64(e), _p64(evk))
        return evk

    def decrypt_coeff(self, c0, c1, s_eval, level: int):
        c0 = np.ascontiguousarray(c0, dtype=np.uint64)
        c1 = np.ascontiguousarray(c1, dtype=np.uint64)
        s = np.ascontiguousarray(s_eval[: level + 1], dtype=np.uint64)
        out = np.empty_like(c0)
        lib().or_decrypt(self._h, _p64(c0), _p64(c1), level, _p64(s), _p64(out))
        return out

    def crt_centered(self, res: np.ndarray, level: int) -> list:
        """Big-int CRT of residues [l+1][N] over q_0..q_l, centered in (-Q/2, Q/2]."""
        qs = self.q[: level + 1]
        Q = 1
        for q in qs:
            Q *= q
        coefs = []
        for i, q in enumerate(qs):
            Qi = Q // q
            coefs.append(Qi * pow(Qi, -1, q))
        out = []
        cols = [[int(v) for v in res[i]] for i in range(level + 1)]
        for x in range(self.n):
            v = 0
            for i in range(level + 1):
                v += cols[i][x] * coefs[i]
            v %= Q
            if v > Q // 2:
                v -= Q
            out.append(v)
        return out


def crt_modulus(primes) -> int:
    Q = 1
    for q in primes:
        Q *= int(q)
    return Q
