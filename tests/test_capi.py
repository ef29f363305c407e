"""CPU tests of the C-ABI boundary: the library loads, exports every symbol include/hks.h declares,
and its host logic (validation, psi, digit layout, workspace sizing) is right.  No compute calls:
a host-only context (device = -1) never touches CUDA."""
import os
import re

import pytest

import hks_synth as S
from conftest import ROOT, read_golden

H = pytest.importorskip("paper_2507_04775_b200.hks")


def header_symbols():
    src = open(os.path.join(ROOT, "include", "hks.h")).read()
    return sorted(set(re.findall(r"\b(hks_[a-z0-9_]+)\s*\(", src)))


def test_exports_match_header():
    lib = H.lib()
    syms = header_symbols()
    assert set(syms) == set(H.EXPORTS)
    for s in syms:
        assert hasattr(lib, s), s


def test_host_ctx_psi_matches_oracle(orc):
    for name in ("C1", "T12", "C2"):
        cfg = S.config(name)
        ctx = H.Context.from_config(cfg, device=-1)
        o = orc.Ctx.from_config(cfg)
        for i in range(len(cfg.q) + len(cfg.p)):
            assert ctx.psi(i) == o.psi(i)


def test_query_digits_golden():
    for L, dnum, level, alpha, sizes in read_golden("digits.txt"):
        L, dnum, level = int(L), int(dnum), int(level)
        primes = S.ntt_primes(10, L + 2, 50)
        ctx = H.Context(10, primes[1:], primes[:1], dnum, device=-1)
        info = ctx.query(level)
        assert info.alpha == int(alpha)
        got = [info.digit_hi[j] - info.digit_lo[j] for j in range(info.beta)]
        assert got == [int(s) for s in sizes.split(",")]


def test_workspace_bytes():
    cfg = S.config("C2")
    ctx = H.Context.from_config(cfg, device=-1)
    lb = cfg.n * 8
    l1, K, ne, beta = 30, 10, 40, 3
    assert ctx.workspace_bytes(H.OP_KEYSWITCH, 29) == (l1 + beta * ne + 2 * ne + 2 * K + 2 * l1) * lb
    assert ctx.workspace_bytes(H.OP_MODUP, 29) == l1 * lb
    assert ctx.workspace_bytes(H.OP_MODDOWN, 9) == (K + 10) * lb
    assert ctx.workspace_bytes(H.OP_KEYSWITCH, 30) == 0       # level > L


def test_validation_errors():
    q = list(S.ntt_primes(12, 4, 50))
    def code(log_n, qq, pp, dnum):
        with pytest.raises(H.HksError) as e:
            H.Context(log_n, qq, pp, dnum, device=-1)
        return e.value.status
    assert code(12, q[1:], [q[0] + 2], 1) in (2, 3)          # not prime or not NTT-friendly
    assert code(12, q[1:], [q[1]], 1) == 5                    # duplicate
    assert code(9, q[1:], q[:1], 1) == 4                      # log_n out of range
    assert code(12, q[1:], q[:1], 4) == 4                     # dnum > L+1
    big = S.ntt_primes(12, 1, 61)[0]
    assert code(12, q[1:], [big], 1) == 4                     # >= 2^60
    p13 = S.ntt_primes(12, 1, 40)[0]                          # 1 mod 2^13 but not 1 mod 2^14
    assert code(13, q[1:], [p13], 1) == 3 or (p13 - 1) % (1 << 14) == 0
    assert code(12, [15], q[:1], 1) == 2                      # composite


def test_host_ctx_refuses_compute():
    cfg = S.config("T10")
    ctx = H.Context.from_config(cfg, device=-1)
    with pytest.raises(H.HksError) as e:
        H.ntt_fwd(ctx, 0x1000, [0], stream=0)
    assert e.value.status == 10


def test_rotate_hoisted_workspace_count_zero_is_worst_case():
    """include/hks.h HKS_OP_ROTATE_HOISTED: count = 0 sizes for every nrot (the layout grows with nrot)."""
    for name, levels in (("C2", (29, 9)), ("T12", (6, 0))):
        cfg = S.config(name)
        ctx = H.Context.from_config(cfg, device=-1)
        for level in levels:
            worst = ctx.workspace_bytes(H.OP_ROTATE_HOISTED, level, 0)
            sizes = [ctx.workspace_bytes(H.OP_ROTATE_HOISTED, level, n) for n in range(1, 65)]
            assert all(a <= b for a, b in zip(sizes, sizes[1:]))          # monotone in nrot
            assert max(sizes) <= worst


def test_bconv_workspace_bytes():
    cfg = S.config("C2")
    ctx = H.Context.from_config(cfg, device=-1)
    lb = cfg.n * 8
    for nsrc, ndst in ((1, 1), (10, 30), (16, 128), (3, 7)):
        b = int(H.lib().hks_bconv_workspace_bytes(ctx.handle, nsrc, ndst))
        assert b >= nsrc * lb + (2 * 16 + nsrc * ndst + ndst * 32 * ((nsrc + 3) // 4)) * 8
        assert b % 128 == 0
    assert int(H.lib().hks_bconv_workspace_bytes(ctx.handle, 17, 4)) == 0      # nsrc > 16
    assert int(H.lib().hks_bconv_workspace_bytes(ctx.handle, 4, 129)) == 0     # ndst > 128
