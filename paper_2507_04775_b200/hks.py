"""Thin ctypes binding of libhks (include/hks.h).  Argument marshalling only: every step of the
hot path runs in the library's CUDA kernels.  torch supplies device memory and streams.

There is no CPU fallback: if libhks.so is missing or a call fails, this module raises.
"""
from __future__ import annotations

import ctypes
import os
from typing import Sequence

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HKS_LIB_PATH") or os.path.join(_HERE, "libhks.so")   # override: experiments only

HKS_OK = 0
STATUS = {0: "HKS_OK", 1: "HKS_EINVAL", 2: "HKS_ENOTPRIME", 3: "HKS_ENOTNTT", 4: "HKS_ERANGE", 5: "HKS_EDUP",
          6: "HKS_EKEY", 7: "HKS_EGALOIS", 8: "HKS_ECUDA", 9: "HKS_ENOMEM", 10: "HKS_EDEVICE"}
OP_MODUP, OP_MODDOWN, OP_KEYSWITCH, OP_ROTATE_HOISTED, OP_HMULT, OP_RESCALE = 0, 1, 2, 3, 4, 5
MAX_DIGITS = 64

# every symbol include/hks.h declares (checked by tests/test_capi.py)
EXPORTS = ("hks_last_error", "hks_ctx_create", "hks_ctx_destroy", "hks_ctx_query", "hks_ctx_psi",
           "hks_workspace_bytes", "hks_ntt_fwd", "hks_ntt_inv", "hks_bconv", "hks_bconv_workspace_bytes", "hks_modup",
           "hks_ksk_inner_product", "hks_moddown", "hks_evk_prepare", "hks_keyswitch", "hks_relinearize", "hks_hmult", "hks_rescale",
           "hks_pt_weighted_sum", "hks_linear_transform", "hks_linear_transform_workspace_bytes",
           "hks_automorph",
           "hks_rotate_hoisted", "hks_rotate_hoisted_batch", "hks_rotate_hoisted_batch_workspace_bytes",
           "hks_launch_count", "hks_prof_enable", "hks_prof_read", "hks_shard_query", "hks_shard_workspace_bytes",
           "hks_shard_ks_modup_in", "hks_shard_ks_inner", "hks_shard_ks_moddown_out", "hks_shard_ks_inner_peer",
           "hks_shard_ks_inner_pipelined", "hks_shard_a2a_query", "hks_shard_a2a_workspace_bytes",
           "hks_shard_a2a_modup_in", "hks_shard_a2a_bconv", "hks_shard_a2a_inner", "hks_shard_a2a_moddown_bconv",
           "hks_shard_a2a_moddown_out",
           "hks_shard_ks_moddown_out_peer")


class HksError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str):
        super().__init__(f"{where}: {STATUS.get(status, status)}: {detail}")
        self.status = status


class ProfEntry(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 32), ("launches", ctypes.c_uint64), ("total_ms", ctypes.c_double),
                ("bytes", ctypes.c_double), ("muls", ctypes.c_double)]


class ShardInfo(ctypes.Structure):
    _fields_ = [(f, ctypes.c_uint32) for f in ("world", "rank", "level", "q_lo", "q_hi", "p_lo", "p_hi", "nq_act",
                                                "q_pad", "p_pad", "nkey")]


class A2AInfo(ctypes.Structure):
    _fields_ = [(f, ctypes.c_uint32) for f in ("chunk_words", "n_pad", "nq_pad", "beta")]


class Info(ctypes.Structure):
    _fields_ = [("log_n", ctypes.c_uint32), ("n", ctypes.c_uint32), ("num_q", ctypes.c_uint32),
                ("num_p", ctypes.c_uint32), ("dnum", ctypes.c_uint32), ("alpha", ctypes.c_uint32),
                ("level", ctypes.c_uint32), ("beta", ctypes.c_uint32),
                ("digit_lo", ctypes.c_uint32 * MAX_DIGITS), ("digit_hi", ctypes.c_uint32 * MAX_DIGITS),
                ("device", ctypes.c_int32)]


_lib = None
_vp = ctypes.c_void_p
_u32 = ctypes.c_uint32
_u64 = ctypes.c_uint64


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2507_04775_b200.build` "
                              "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        L.hks_last_error.restype = ctypes.c_char_p
        L.hks_ctx_create.argtypes = [_u32, ctypes.POINTER(_u64), _u32, ctypes.POINTER(_u64), _u32, _u32,
                                     ctypes.c_int, ctypes.POINTER(_vp)]
        L.hks_ctx_destroy.argtypes = [_vp]
        L.hks_ctx_destroy.restype = None
        L.hks_ctx_query.argtypes = [_vp, _u32, ctypes.POINTER(Info)]
        L.hks_ctx_psi.argtypes = [_vp, _u32, ctypes.POINTER(_u64)]
        L.hks_workspace_bytes.argtypes = [_vp, ctypes.c_int, _u32, _u32]
        L.hks_workspace_bytes.restype = ctypes.c_size_t
        for f in ("hks_ntt_fwd", "hks_ntt_inv"):
            getattr(L, f).argtypes = [_vp, _vp, ctypes.POINTER(_u32), _u32, _vp]
        L.hks_bconv.argtypes = [_vp, _vp, ctypes.POINTER(_u32), _u32, ctypes.POINTER(_u32), _u32, _vp, _vp, _vp]
        L.hks_bconv_workspace_bytes.argtypes = [_vp, _u32, _u32]
        L.hks_bconv_workspace_bytes.restype = ctypes.c_size_t
        L.hks_modup.argtypes = [_vp, _vp, _u32, _vp, _vp, _vp]
        L.hks_ksk_inner_product.argtypes = [_vp, _vp, _vp, _u32, _u32, _u64, _vp, _vp]
        L.hks_moddown.argtypes = [_vp, _vp, _u32, _vp, _vp, _vp]
        L.hks_keyswitch.argtypes = [_vp, _vp, _vp, _u32, _vp, _u32, _vp, _vp, _vp, _vp]
        L.hks_evk_prepare.argtypes = [_vp, _vp, _u32, _vp, _vp]
        L.hks_automorph.argtypes = [_vp, _vp, _u32, _u64, _vp, _vp]
        L.hks_relinearize.argtypes = [_vp, _vp, _vp, _vp, _u32, _vp, _u32, _vp, _vp, _vp, _vp]
        L.hks_hmult.argtypes = [_vp, _vp, _vp, _vp, _vp, _u32, _vp, _u32, _vp, _vp, _vp, _vp]
        L.hks_rescale.argtypes = [_vp, _vp, _u32, _u32, _vp, _vp, _vp]
        _vpp = ctypes.POINTER(_vp)
        L.hks_pt_weighted_sum.argtypes = [_vp, _u32, _vpp, _vpp, _vpp, _u32, _vp, _vp, _vp]
        L.hks_linear_transform.argtypes = [_vp, _vp, _vp, _u32, _u32, _u32, ctypes.POINTER(_u64), _vpp,
                                           ctypes.POINTER(_u64), _vpp, _u32, _vpp, _vp, _vp, _vp, _vp]
        L.hks_linear_transform_workspace_bytes.restype = ctypes.c_size_t
        L.hks_linear_transform_workspace_bytes.argtypes = [_vp, _u32, _u32]
        L.hks_rotate_hoisted.argtypes = [_vp, _vp, _vp, _u32, _u32, ctypes.POINTER(_u64), ctypes.POINTER(_vp), _u32,
                                         ctypes.POINTER(_vp), ctypes.POINTER(_vp), _vp, _vp]
        L.hks_launch_count.restype = ctypes.c_uint64
        L.hks_launch_count.argtypes = []
        L.hks_prof_enable.argtypes = [ctypes.c_int]
        L.hks_prof_read.argtypes = [ctypes.POINTER(ProfEntry), ctypes.c_int]
        L.hks_rotate_hoisted_batch.argtypes = [_vp, _u32, ctypes.POINTER(_vp), ctypes.POINTER(_vp), _u32, _u32,
                                               ctypes.POINTER(_u64), ctypes.POINTER(_vp), _u32, ctypes.POINTER(_vp),
                                               ctypes.POINTER(_vp), _vp, _vp]
        L.hks_rotate_hoisted_batch_workspace_bytes.argtypes = [_vp, _u32, _u32]
        L.hks_rotate_hoisted_batch_workspace_bytes.restype = ctypes.c_size_t
        L.hks_shard_query.argtypes = [_vp, _u32, _u32, _u32, ctypes.POINTER(ShardInfo)]
        L.hks_shard_workspace_bytes.argtypes = [_vp, _u32, _u32, _u32]
        L.hks_shard_workspace_bytes.restype = ctypes.c_size_t
        L.hks_shard_ks_modup_in.argtypes = [_vp, _u32, _u32, _u32, _vp, _vp, _vp]
        L.hks_shard_ks_inner.argtypes = [_vp, _u32, _u32, _u32, _vp, _vp, _vp, _u32, _vp, _vp, _vp, _vp]
        L.hks_shard_ks_moddown_out.argtypes = [_vp, _u32, _u32, _u32, _vp, _vp, _vp, _vp, _vp, _vp, _vp]
        L.hks_shard_ks_inner_pipelined.argtypes = [_vp, _u32, _u32, _u32, _vp, ctypes.POINTER(_vp), _vp, _vp, _u32, _vp,
                                                   _vp, _vp, _vp]
        L.hks_shard_a2a_query.argtypes = [_vp, _u32, _u32, _u32, ctypes.POINTER(A2AInfo)]
        L.hks_shard_a2a_workspace_bytes.argtypes = [_vp, _u32, _u32, _u32]
        L.hks_shard_a2a_workspace_bytes.restype = ctypes.c_size_t
        L.hks_shard_a2a_modup_in.argtypes = [_vp, _u32, _u32, _u32, _vp, _vp, _vp, _vp]
        L.hks_shard_a2a_bconv.argtypes = [_vp, _u32, _u32, _u32, _vp, _vp, _vp]
        L.hks_shard_a2a_inner.argtypes = [_vp, _u32, _u32, _u32, _vp, _vp, _vp, _u32, _vp, _vp, _vp, _vp]
        L.hks_shard_a2a_moddown_bconv.argtypes = [_vp, _u32, _u32, _u32, _vp, _vp, _vp]
        L.hks_shard_a2a_moddown_out.argtypes = [_vp, _u32, _u32, _u32, _vp, _vp, _vp, _vp, _vp, _vp, _vp]
        L.hks_shard_ks_inner_peer.argtypes = [_vp, _u32, _u32, _u32, ctypes.POINTER(_vp), _vp, _vp, _u32, _vp, _vp,
                                              _vp, _vp]
        L.hks_shard_ks_moddown_out_peer.argtypes = [_vp, _u32, _u32, _u32, ctypes.POINTER(_vp), _vp, _vp, _vp, _vp,
                                                    _vp, _vp]
        for f in EXPORTS[1:]:
            if f not in ("hks_ctx_destroy", "hks_workspace_bytes", "hks_launch_count", "hks_shard_workspace_bytes",
                         "hks_rotate_hoisted_batch_workspace_bytes", "hks_bconv_workspace_bytes",
                         "hks_shard_a2a_workspace_bytes",
                         "hks_linear_transform_workspace_bytes"):
                getattr(L, f).restype = ctypes.c_int
        _lib = L
    return _lib


def _check(st: int, where: str):
    if st != HKS_OK:
        raise HksError(st, where, lib().hks_last_error().decode())


def _u32arr(seq: Sequence[int]):
    return (_u32 * len(seq))(*[int(v) for v in seq])


def _ptr(t) -> int:
    """Device pointer of a torch tensor (or a raw int / None)."""
    if t is None:
        return None
    if isinstance(t, int):
        return t
    return t.data_ptr()


HKS_EVK_PREPARED = 0x10000   # include/hks.h: evk_digits flag of a key from hks_evk_prepare


class PreparedKey:
    """A key returned by evk_prepare: the device tensor [digits][2][L+1+K][N] and the flag every key-taking call
    passes with its digit count (HKS_EVK_PREPARED)."""

    def __init__(self, tensor):
        self.tensor = tensor
        self.shape = tensor.shape

    def data_ptr(self) -> int:
        return self.tensor.data_ptr()


def evk_digits(ctx, evk) -> int:
    """Digit count of a key passed to libhks: the leading dimension of a [digits][2][L+1+K][N] tensor, or
    of the first of a list of keys; a raw address carries none, so the context's dnum is assumed.  A
    PreparedKey (or a list of them) adds HKS_EVK_PREPARED."""
    if isinstance(evk, (list, tuple)):
        flags = {isinstance(e, PreparedKey) for e in evk}
        if len(flags) > 1:
            raise ValueError("hks: a call takes either prepared keys or plain keys, not both")
        return min((evk_digits(ctx, e) for e in evk), default=ctx.dnum)
    shape = getattr(evk, "shape", None)
    d = int(shape[0]) if shape is not None and len(shape) == 4 else ctx.dnum
    return d | HKS_EVK_PREPARED if isinstance(evk, PreparedKey) else d


def evk_prepare(ctx: "Context", evk, out=None, stream=None) -> PreparedKey:
    """hks_evk_prepare: the key's Q limbs times P^-1 (in place when out is None or out is evk)."""
    dst = evk if out is None else out
    _check(lib().hks_evk_prepare(ctx.handle, _ptr(evk), evk_digits(ctx, evk), _ptr(dst), _stream(stream)),
           "hks_evk_prepare")
    return PreparedKey(dst)


def _stream(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


class Context:
    """hks_ctx handle: (N = 2^log_n, q chain, special primes p, dnum) on `device` (-1: host-only)."""

    def __init__(self, log_n: int, q: Sequence[int], p: Sequence[int], dnum: int, device: int = 0):
        qa = (_u64 * len(q))(*[int(v) for v in q])
        pa = (_u64 * len(p))(*[int(v) for v in p])
        h = _vp()
        _check(lib().hks_ctx_create(log_n, qa, len(q), pa, len(p), dnum, device, ctypes.byref(h)), "hks_ctx_create")
        self._h = h
        self.log_n, self.n = log_n, 1 << log_n
        self.q, self.p, self.dnum, self.device = tuple(q), tuple(p), dnum, device
        self.nq, self.np = len(q), len(p)
        self.alpha = -(-self.nq // dnum)

    @classmethod
    def from_config(cls, cfg, device: int = 0):
        return cls(cfg.log_n, cfg.q, cfg.p, cfg.dnum, device)

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None):
            lib().hks_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def query(self, level: int) -> Info:
        info = Info()
        _check(lib().hks_ctx_query(self._h, level, ctypes.byref(info)), "hks_ctx_query")
        return info

    def psi(self, prime_idx: int) -> int:
        v = _u64()
        _check(lib().hks_ctx_psi(self._h, prime_idx, ctypes.byref(v)), "hks_ctx_psi")
        return int(v.value)

    def workspace_bytes(self, op: int, level: int, count: int = 0) -> int:
        return int(lib().hks_workspace_bytes(self._h, op, level, count))

    def beta(self, level: int) -> int:
        return -(-(level + 1) // self.alpha)

    def workspace(self, op: int, level: int, count: int = 0):
        import torch
        nbytes = self.workspace_bytes(op, level, count)
        return torch.empty(max(nbytes // 8, 1), dtype=torch.uint64, device=f"cuda:{self.device}")


def ntt_fwd(ctx: Context, x, prime_idx: Sequence[int], stream=None):
    _check(lib().hks_ntt_fwd(ctx.handle, _ptr(x), _u32arr(prime_idx), len(prime_idx), _stream(stream)), "hks_ntt_fwd")


def ntt_inv(ctx: Context, x, prime_idx: Sequence[int], stream=None):
    _check(lib().hks_ntt_inv(ctx.handle, _ptr(x), _u32arr(prime_idx), len(prime_idx), _stream(stream)), "hks_ntt_inv")


def bconv_workspace(ctx: Context, nsrc: int, ndst: int):
    import torch
    nbytes = int(lib().hks_bconv_workspace_bytes(ctx.handle, nsrc, ndst))
    return torch.empty(max(nbytes // 8, 1), dtype=torch.uint64, device=f"cuda:{ctx.device}")


def bconv(ctx: Context, x, src_idx: Sequence[int], dst_idx: Sequence[int], out, ws=None, stream=None):
    """ws: bconv_workspace(ctx, len(src_idx), len(dst_idx)) (allocated here when None)."""
    if ws is None:
        ws = bconv_workspace(ctx, len(src_idx), len(dst_idx))
    _check(lib().hks_bconv(ctx.handle, _ptr(x), _u32arr(src_idx), len(src_idx), _u32arr(dst_idx), len(dst_idx),
                           _ptr(out), _ptr(ws), _stream(stream)), "hks_bconv")


def modup(ctx: Context, d, level: int, ext, ws, stream=None):
    _check(lib().hks_modup(ctx.handle, _ptr(d), level, _ptr(ext), _ptr(ws), _stream(stream)), "hks_modup")


def ksk_inner_product(ctx: Context, ext, evk, level: int, galois: int, acc, stream=None):
    _check(lib().hks_ksk_inner_product(ctx.handle, _ptr(ext), _ptr(evk), evk_digits(ctx, evk), level, galois, _ptr(acc),
                                       _stream(stream)),
           "hks_ksk_inner_product")


def moddown(ctx: Context, acc, level: int, out, ws, stream=None):
    _check(lib().hks_moddown(ctx.handle, _ptr(acc), level, _ptr(out), _ptr(ws), _stream(stream)), "hks_moddown")


def keyswitch(ctx: Context, c0, c1, level: int, evk, out0, out1, ws, stream=None):
    _check(lib().hks_keyswitch(ctx.handle, _ptr(c0), _ptr(c1), level, _ptr(evk), evk_digits(ctx, evk), _ptr(out0),
                               _ptr(out1), _ptr(ws), _stream(stream)), "hks_keyswitch")


def relinearize(ctx: Context, d0, d1, d2, level: int, evk, out0, out1, ws, stream=None):
    _check(lib().hks_relinearize(ctx.handle, _ptr(d0), _ptr(d1), _ptr(d2), level, _ptr(evk), evk_digits(ctx, evk),
                                 _ptr(out0), _ptr(out1), _ptr(ws), _stream(stream)), "hks_relinearize")


def hmult(ctx: Context, a0, a1, b0, b1, level: int, evk, out0, out1, ws, stream=None):
    _check(lib().hks_hmult(ctx.handle, _ptr(a0), _ptr(a1), _ptr(b0), _ptr(b1), level, _ptr(evk), evk_digits(ctx, evk),
                           _ptr(out0), _ptr(out1), _ptr(ws), _stream(stream)), "hks_hmult")


def rescale(ctx: Context, x, npoly: int, level: int, out, ws, stream=None):
    _check(lib().hks_rescale(ctx.handle, _ptr(x), npoly, level, _ptr(out), _ptr(ws), _stream(stream)), "hks_rescale")


def pt_weighted_sum(ctx: Context, w, x0, x1, level: int, out0, out1, stream=None):
    n = len(w)
    arr = lambda vs: (_vp * n)(*[_ptr(v) for v in vs])
    _check(lib().hks_pt_weighted_sum(ctx.handle, n, arr(w), arr(x0), arr(x1), level, _ptr(out0), _ptr(out1),
                                     _stream(stream)), "hks_pt_weighted_sum")


def linear_transform_workspace(ctx: Context, level: int, n1: int):
    import torch
    nbytes = int(lib().hks_linear_transform_workspace_bytes(ctx.handle, level, n1))
    return torch.empty(max(nbytes // 8, 1), dtype=torch.uint64, device=f"cuda:{ctx.device}")


def linear_transform(ctx: Context, c0, c1, level: int, n1: int, n2: int, baby_galois, baby_evks, giant_galois,
                     giant_evks, pts, out0, out1, ws, stream=None):
    """pts: n1*n2 diagonals (index i*n1 + j); baby lists n1-1 entries, giant lists n2-1 entries."""
    arr = lambda vs: (_vp * max(1, len(vs)))(*[_ptr(v) for v in vs])
    gal = lambda vs: (_u64 * max(1, len(vs)))(*[int(v) for v in vs])
    _check(lib().hks_linear_transform(ctx.handle, _ptr(c0), _ptr(c1), level, n1, n2, gal(baby_galois), arr(baby_evks),
                                      gal(giant_galois), arr(giant_evks), evk_digits(ctx, list(baby_evks) + list(giant_evks)),
                                      arr(pts), _ptr(out0), _ptr(out1), _ptr(ws), _stream(stream)), "hks_linear_transform")


def automorph(ctx: Context, x, nlimbs: int, galois: int, out, stream=None):
    _check(lib().hks_automorph(ctx.handle, _ptr(x), nlimbs, galois, _ptr(out), _stream(stream)), "hks_automorph")


def rotate_hoisted(ctx: Context, c0, c1, level: int, galois: Sequence[int], evks, outs0, outs1, ws, stream=None):
    n = len(galois)
    g = (_u64 * n)(*[int(v) for v in galois])
    ek = (_vp * n)(*[_ptr(e) for e in evks])
    o0 = (_vp * n)(*[_ptr(o) for o in outs0])
    o1 = (_vp * n)(*[_ptr(o) for o in outs1])
    _check(lib().hks_rotate_hoisted(ctx.handle, _ptr(c0), _ptr(c1), level, n, g, ek, evk_digits(ctx, list(evks)), o0, o1,
                                    _ptr(ws), _stream(stream)), "hks_rotate_hoisted")


def launch_count() -> int:
    """Kernels libhks has launched in this process."""
    return int(lib().hks_launch_count())


def prof_enable(on: bool = True):
    _check(lib().hks_prof_enable(1 if on else 0), "hks_prof_enable")


def prof_read() -> dict:
    """{kernel class: (launches, total_ms, algorithmic_bytes, algorithmic_muls)} since the last read."""
    arr = (ProfEntry * 16)()
    k = lib().hks_prof_read(arr, 16)
    return {arr[i].name.decode(): (int(arr[i].launches), float(arr[i].total_ms), float(arr[i].bytes),
                                   float(arr[i].muls)) for i in range(k)}


def rotate_hoisted_batch(ctx: Context, c0s, c1s, level: int, galois: Sequence[int], evks, outs0, outs1, ws,
                         stream=None):
    """outs0/outs1: flat lists, index ct * nrot + r."""
    nct, n = len(c0s), len(galois)
    g = (_u64 * n)(*[int(v) for v in galois])
    a0 = (_vp * nct)(*[_ptr(x) for x in c0s])
    a1 = (_vp * nct)(*[_ptr(x) for x in c1s])
    ek = (_vp * n)(*[_ptr(e) for e in evks])
    o0 = (_vp * (nct * n))(*[_ptr(o) for o in outs0])
    o1 = (_vp * (nct * n))(*[_ptr(o) for o in outs1])
    _check(lib().hks_rotate_hoisted_batch(ctx.handle, nct, a0, a1, level, n, g, ek, evk_digits(ctx, list(evks)), o0, o1,
                                          _ptr(ws), _stream(stream)),
           "hks_rotate_hoisted_batch")


def rotate_hoisted_batch_workspace(ctx: Context, nct: int, level: int):
    import torch
    nbytes = int(lib().hks_rotate_hoisted_batch_workspace_bytes(ctx.handle, nct, level))
    return torch.empty(max(nbytes // 8, 1), dtype=torch.uint64, device=f"cuda:{ctx.device}")


# ---- limb-sharded KeySwitch (C4): phases of include/hks.h; the all-gathers are the caller's
def shard_query(ctx: Context, level: int, world: int, rank: int) -> ShardInfo:
    info = ShardInfo()
    _check(lib().hks_shard_query(ctx.handle, level, world, rank, ctypes.byref(info)), "hks_shard_query")
    return info


def shard_workspace_bytes(ctx: Context, level: int, world: int, rank: int) -> int:
    return int(lib().hks_shard_workspace_bytes(ctx.handle, level, world, rank))


def shard_ks_modup_in(ctx: Context, level, world, rank, c1_loc, ysend, stream=None):
    _check(lib().hks_shard_ks_modup_in(ctx.handle, level, world, rank, _ptr(c1_loc), _ptr(ysend), _stream(stream)),
           "hks_shard_ks_modup_in")


def shard_ks_inner(ctx: Context, level, world, rank, yall, c1_loc, evk_loc, acc_loc, ypsend, ws, stream=None):
    _check(lib().hks_shard_ks_inner(ctx.handle, level, world, rank, _ptr(yall), _ptr(c1_loc), _ptr(evk_loc),
                                    evk_digits(ctx, evk_loc), _ptr(acc_loc), _ptr(ypsend), _ptr(ws), _stream(stream)),
           "hks_shard_ks_inner")


def shard_ks_inner_pipelined(ctx: Context, level, world, rank, yall, digit_events, c1_loc, evk_loc, acc_loc, ypsend,
                             ws, stream=None):
    """Phase B with one base-conversion launch per digit, digit j after `stream` waits on digit_events[j]
    (torch.cuda.Event, raw cudaEvent_t int, or None)."""
    ev = [None if e is None else (e if isinstance(e, int) else e.cuda_event) for e in digit_events]
    arr = (_vp * max(1, len(ev)))(*ev)
    _check(lib().hks_shard_ks_inner_pipelined(ctx.handle, level, world, rank, _ptr(yall), arr, _ptr(c1_loc),
                                              _ptr(evk_loc), evk_digits(ctx, evk_loc), _ptr(acc_loc), _ptr(ypsend),
                                              _ptr(ws), _stream(stream)), "hks_shard_ks_inner_pipelined")


def _ptr_table(ptrs):
    """HOST array of device addresses (ints or tensors) for the *_peer phases."""
    vals = [p if isinstance(p, int) else _ptr(p) for p in ptrs]
    return (_vp * len(vals))(*vals)


def shard_ks_inner_peer(ctx: Context, level, world, rank, ysend_ranks, c1_loc, evk_loc, acc_loc, ypsend, ws,
                        stream=None):
    """Phase B reading every rank's ysend through `ysend_ranks` (addresses valid on this GPU: own buffer,
    peer mappings over NVLink, or simulated ranks' buffers on one device) -- no all-gather."""
    _check(lib().hks_shard_ks_inner_peer(ctx.handle, level, world, rank, _ptr_table(ysend_ranks), _ptr(c1_loc),
                                         _ptr(evk_loc), evk_digits(ctx, evk_loc), _ptr(acc_loc), _ptr(ypsend), _ptr(ws),
                                         _stream(stream)),
           "hks_shard_ks_inner_peer")


def shard_ks_moddown_out_peer(ctx: Context, level, world, rank, ypsend_ranks, acc_loc, c0_loc, out0_loc, out1_loc,
                              ws, stream=None):
    _check(lib().hks_shard_ks_moddown_out_peer(ctx.handle, level, world, rank, _ptr_table(ypsend_ranks),
                                               _ptr(acc_loc), _ptr(c0_loc), _ptr(out0_loc), _ptr(out1_loc),
                                               _ptr(ws), _stream(stream)), "hks_shard_ks_moddown_out_peer")


def shard_ks_moddown_out(ctx: Context, level, world, rank, ypall, acc_loc, c0_loc, out0_loc, out1_loc, ws,
                         stream=None):
    _check(lib().hks_shard_ks_moddown_out(ctx.handle, level, world, rank, _ptr(ypall), _ptr(acc_loc), _ptr(c0_loc),
                                          _ptr(out0_loc), _ptr(out1_loc), _ptr(ws), _stream(stream)),
           "hks_shard_ks_moddown_out")


# ---- all-to-all coefficient-sharded KeySwitch (include/hks.h "All-to-all coefficient-sharded KeySwitch")
def shard_a2a_query(ctx: Context, level: int, world: int, rank: int) -> A2AInfo:
    info = A2AInfo()
    _check(lib().hks_shard_a2a_query(ctx.handle, level, world, rank, ctypes.byref(info)), "hks_shard_a2a_query")
    return info


def shard_a2a_workspace_bytes(ctx: Context, level: int, world: int, rank: int) -> int:
    return int(lib().hks_shard_a2a_workspace_bytes(ctx.handle, level, world, rank))


def shard_a2a_modup_in(ctx: Context, level, world, rank, c1_loc, ysend, ws, stream=None):
    _check(lib().hks_shard_a2a_modup_in(ctx.handle, level, world, rank, _ptr(c1_loc), _ptr(ysend), _ptr(ws),
                                        _stream(stream)), "hks_shard_a2a_modup_in")


def shard_a2a_bconv(ctx: Context, level, world, rank, yrecv, extsend, stream=None):
    _check(lib().hks_shard_a2a_bconv(ctx.handle, level, world, rank, _ptr(yrecv), _ptr(extsend), _stream(stream)),
           "hks_shard_a2a_bconv")


def shard_a2a_inner(ctx: Context, level, world, rank, extrecv, c1_loc, evk_loc, acc_loc, ypsend, ws, stream=None):
    _check(lib().hks_shard_a2a_inner(ctx.handle, level, world, rank, _ptr(extrecv), _ptr(c1_loc), _ptr(evk_loc),
                                     evk_digits(ctx, evk_loc), _ptr(acc_loc), _ptr(ypsend), _ptr(ws), _stream(stream)),
           "hks_shard_a2a_inner")


def shard_a2a_moddown_bconv(ctx: Context, level, world, rank, yprecv, convsend, stream=None):
    _check(lib().hks_shard_a2a_moddown_bconv(ctx.handle, level, world, rank, _ptr(yprecv), _ptr(convsend),
                                             _stream(stream)), "hks_shard_a2a_moddown_bconv")


def shard_a2a_moddown_out(ctx: Context, level, world, rank, convrecv, acc_loc, c0_loc, out0_loc, out1_loc, ws,
                          stream=None):
    _check(lib().hks_shard_a2a_moddown_out(ctx.handle, level, world, rank, _ptr(convrecv), _ptr(acc_loc),
                                           _ptr(c0_loc), _ptr(out0_loc), _ptr(out1_loc), _ptr(ws), _stream(stream)),
           "hks_shard_a2a_moddown_out")
