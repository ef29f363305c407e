"""GPU parity: every hot-path step through the C ABI, bit-exact against the CPU oracle on the same
seeded inputs (integer arithmetic -> the bar is bit-exact; BASELINE.json north_star).

Sizes: small rings (several tiles, ragged digits, partial digits at lower levels) for every
function, and the full BASELINE.json configurations (C1, C2 at N=2^16/L=29/dnum=3, C4 at
N=2^17/L=35/dnum=4) in the same launch configuration bench.py times."""
import numpy as np
import pytest

import hks_synth as S
from helpers import Keys, empty_dev, encrypt_under, ks_bound, to_dev, to_host

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
H = pytest.importorskip("paper_2507_04775_b200.hks")


@pytest.fixture(autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


_CTX = {}


def ctxs(orc, name):
    if name not in _CTX:
        cfg = S.config(name)
        _CTX[name] = (cfg, H.Context.from_config(cfg, 0), orc.Ctx.from_config(cfg))
    return _CTX[name]


def edge_limbs(primes, n, g):
    x = S.uniform_limbs(g, primes, n)
    for b, p in enumerate(primes):
        x[b, :8] = [0, 1, p - 1, p - 2, 2, 0, p - 1, 1]
    return x


# ------------------------------------------------------------------ NTT

@pytest.mark.parametrize("log_n", [10, 11, 12, 13, 14, 15, 16, 17])
def test_ntt_parity(orc, log_n):
    primes = S.ntt_primes(log_n, 5, 60)
    q, p = primes[1:], primes[:1]
    ctx = H.Context(log_n, q, p, 1, 0)
    o = orc.Ctx(log_n, q, p, 1)
    g = S.rng(400 + log_n)
    idx = [0, 1, 2, 3, 4, 2, 0]
    x = edge_limbs([o.primes[i] for i in idx], o.n, g)
    d = to_dev(x)
    H.ntt_fwd(ctx, d, idx)
    want = o.ntt(x, idx)
    got = to_host(d)
    assert (got == want).all()
    H.ntt_inv(ctx, d, idx)
    assert (to_host(d) == x).all()
    y = to_dev(want)
    H.ntt_inv(ctx, y, idx)
    assert (to_host(y) == o.intt(want, idx)).all()


def test_ntt_batch_invariance(orc):
    cfg, ctx, o = ctxs(orc, "T16s")
    g = S.rng(410)
    idx = list(range(len(o.primes))) * 3
    x = S.uniform_limbs(g, [o.primes[i] for i in idx], o.n)
    d = to_dev(x)
    H.ntt_fwd(ctx, d, idx)
    whole = to_host(d)
    for b in range(len(idx)):
        e = to_dev(x[b:b + 1])
        H.ntt_fwd(ctx, e, [idx[b]])
        assert (to_host(e)[0] == whole[b]).all()


def test_ntt_large_batch(orc):
    # more limbs than one launch carries (HKS_MAXB = 256)
    primes = S.ntt_primes(10, 3, 60)
    ctx = H.Context(10, primes[1:], primes[:1], 1, 0)
    o = orc.Ctx(10, primes[1:], primes[:1], 1)
    g = S.rng(411)
    idx = [i % 3 for i in range(300)]
    x = S.uniform_limbs(g, [o.primes[i] for i in idx], o.n)
    d = to_dev(x)
    H.ntt_fwd(ctx, d, idx)
    assert (to_host(d) == o.ntt(x, idx)).all()


# ------------------------------------------------------------------ BConv, automorphism

@pytest.mark.parametrize("name,src,dst", [("T12", [0, 1, 2], [3, 4, 5, 6, 7, 8, 9]),
                                          ("C2", list(range(10)), list(range(10, 40))),
                                          ("C2", list(range(30, 40)), list(range(30))),
                                          ("T12", [5], [0, 1, 9]),
                                          ("C4", list(range(36, 45)), list(range(36))),
                                          ("C4", [7], list(range(7)) + list(range(8, 45))),
                                          ("C1", [0, 1, 2], [3]),
                                          ("C2", list(range(10)), list(range(10, 39))),
                                          ("C2", [3, 17, 25], [0, 1, 2, 39, 38, 37, 10]),
                                          ("C4", list(range(16)), list(range(16, 45)))])
def test_bconv_parity(orc, name, src, dst):
    cfg, ctx, o = ctxs(orc, name)
    g = S.rng(420)
    x = edge_limbs([o.primes[i] for i in src], o.n, g)
    out = empty_dev((len(dst), o.n))
    H.bconv(ctx, to_dev(x), src, dst, out)
    assert (to_host(out) == o.bconv(x, src, dst)).all()


@pytest.mark.parametrize("name", ["T12", "C2"])
def test_automorph_parity(orc, name):
    cfg, ctx, o = ctxs(orc, name)
    g = S.rng(430)
    x = S.uniform_limbs(g, o.primes[:4], o.n)
    for k in (S.galois_rot(1, cfg.log_n), S.galois_rot(7, cfg.log_n), S.GALOIS_CONJ(cfg.log_n)):
        out = empty_dev((4, o.n))
        H.automorph(ctx, to_dev(x), 4, k, out)
        assert (to_host(out) == o.automorph(x, k)).all()


# ------------------------------------------------------------------ ModUp, KIP, ModDown

@pytest.mark.parametrize("name,level", [("T12", 6), ("T12", 3), ("T12", 0), ("C2", 29), ("C2", 20), ("C2", 9)])
def test_modup_parity(orc, name, level):
    cfg, ctx, o = ctxs(orc, name)
    g = S.rng(440 + level)
    d = edge_limbs(o.q[: level + 1], o.n, g)
    beta = ctx.beta(level)
    ne = level + 1 + o.np
    ext = empty_dev((beta, ne, o.n))
    ws = ctx.workspace(H.OP_MODUP, level)
    H.modup(ctx, to_dev(d), level, ext, ws)
    assert (to_host(ext) == o.modup(d, level)).all()


@pytest.mark.parametrize("name,level,galois", [("T12", 6, 1), ("T12", 4, 5), ("C2", 29, 1), ("C2", 15, 25)])
def test_kip_parity(orc, name, level, galois):
    cfg, ctx, o = ctxs(orc, name)
    g = S.rng(450 + level)
    beta = ctx.beta(level)
    eidx = o.ext_primes(level)
    ext = np.stack([S.uniform_limbs(g, [o.primes[i] for i in eidx], o.n) for _ in range(beta)])
    nk = o.nq + o.np
    evk = np.stack([S.uniform_limbs(g, o.primes, o.n) for _ in range(2 * o.dnum)]).reshape(o.dnum, 2, nk, o.n)
    acc = empty_dev((2, len(eidx), o.n))
    H.ksk_inner_product(ctx, to_dev(ext), to_dev(evk), level, galois, acc)
    assert (to_host(acc) == o.kip(ext, evk, level, galois)).all()


@pytest.mark.parametrize("name,level", [("T12", 6), ("T12", 1), ("C2", 29), ("C2", 9), ("C2", 0)])
def test_moddown_parity(orc, name, level):
    cfg, ctx, o = ctxs(orc, name)
    g = S.rng(460 + level)
    eidx = o.ext_primes(level)
    acc = edge_limbs([o.primes[i] for i in eidx], o.n, g)
    out = empty_dev((level + 1, o.n))
    ws = ctx.workspace(H.OP_MODDOWN, level)
    H.moddown(ctx, to_dev(acc), level, out, ws)
    assert (to_host(out) == o.moddown(acc, level)).all()


# ------------------------------------------------------------------ KeySwitch end to end

_KEYS = {}


def relin_key(o, name):
    if name not in _KEYS:
        cfg = S.config(name)
        k = Keys(o, cfg.seed)
        _KEYS[name] = (k, k.relin())
    return _KEYS[name]


def run_ks(ctx, c0, c1, level, evk_dev):
    out0 = empty_dev(c0.shape)
    out1 = empty_dev(c1.shape)
    ws = ctx.workspace(H.OP_KEYSWITCH, level)
    H.keyswitch(ctx, to_dev(c0), to_dev(c1), level, evk_dev, out0, out1, ws)
    return to_host(out0), to_host(out1)


@pytest.mark.parametrize("name,levels", [("C1", [2]), ("C1p", [2, 1, 0]), ("T10", [4, 2]),
                                         ("T12", [6, 5, 4, 3, 0]), ("T16s", [5, 1]), ("T17s", [4])])
def test_keyswitch_parity_small(orc, name, levels):
    cfg, ctx, o = ctxs(orc, name)
    keys, evk = relin_key(o, name)
    evk_d = to_dev(evk)
    s2 = o.mul(keys.s_eval, keys.s_eval, list(range(keys.nk)))
    g = S.rng(cfg.seed + 7)
    for level in levels:
        m, c0, c1 = encrypt_under(o, g, s2, level, 20)
        got0, got1 = run_ks(ctx, c0, c1, level, evk_d)
        want0, want1 = o.keyswitch(c0, c1, evk, level)
        assert (got0 == want0).all() and (got1 == want1).all(), level
        dec = o.crt_centered(o.decrypt_coeff(got0, got1, keys.s_eval, level), level)
        err = max(abs(a - int(b)) for a, b in zip(dec, m))
        assert err <= ks_bound(o, level, keys.B_e, keys.h)


def test_evk_digit_count(orc):
    """include/hks.h "Keys" / SPEC.md:482: a key with fewer digits than beta(level) is refused with HKS_EKEY
    before any launch; the same key is usable (bit-exact) at a level it covers."""
    cfg, ctx, o = ctxs(orc, "C2")
    keys, evk = relin_key(o, "C2")
    g = S.rng(cfg.seed + 77)
    short = to_dev(np.ascontiguousarray(evk[:2]))          # 2 of 3 digits: covers levels <= 19
    level = 29
    c0, c1 = (S.uniform_limbs(g, o.q[: level + 1], o.n) for _ in range(2))
    out0, out1 = empty_dev(c0.shape), empty_dev(c0.shape)
    ws = ctx.workspace(H.OP_KEYSWITCH, level)
    with pytest.raises(H.HksError) as ei:
        H.keyswitch(ctx, to_dev(c0), to_dev(c1), level, short, out0, out1, ws)
    assert ei.value.status == 6
    with pytest.raises(H.HksError) as ei:
        H.hmult(ctx, to_dev(c0), to_dev(c1), to_dev(c0), to_dev(c1), level, short, out0, out1,
                ctx.workspace(H.OP_HMULT, level))
    assert ei.value.status == 6
    level = 19
    c0, c1 = c0[: level + 1], c1[: level + 1]
    got0, got1 = run_ks(ctx, c0, c1, level, short)
    want0, want1 = o.keyswitch(c0, c1, evk, level)
    assert (got0 == want0).all() and (got1 == want1).all()


def test_bconv_graph_capture(orc):
    """hks_bconv derives its constants on the device into the caller's workspace: no allocation and no host
    copy inside the call, so it can be captured into a CUDA graph; the replays are bit-exact."""
    cfg, ctx, o = ctxs(orc, "C2")
    src, dst = [3, 17, 25, 31], [0, 1, 2, 39, 38, 37, 10]
    g = S.rng(421)
    xs = [edge_limbs([o.primes[i] for i in src], o.n, g) for _ in range(2)]
    x = to_dev(xs[0])
    out = empty_dev((len(dst), o.n))
    ws = H.bconv_workspace(ctx, len(src), len(dst))
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        H.bconv(ctx, x, src, dst, out, ws, torch.cuda.current_stream().cuda_stream)
    for xv in xs:
        x.copy_(to_dev(xv))
        gr.replay()
        torch.cuda.synchronize()
        assert (to_host(out) == o.bconv(xv, src, dst)).all()


@pytest.mark.parametrize("level", [29, 27, 20, 19, 11, 9, 0])
def test_keyswitch_parity_c2(orc, level):
    """BASELINE.json configs[1]: N=2^16, L=29, dnum=3, 60-bit primes; level sweep across digit drops."""
    cfg, ctx, o = ctxs(orc, "C2")
    keys, evk = relin_key(o, "C2")
    g = S.rng(cfg.seed + 100 + level)
    c0 = S.uniform_limbs(g, o.q[: level + 1], o.n)
    c1 = edge_limbs(o.q[: level + 1], o.n, g)
    got0, got1 = run_ks(ctx, c0, c1, level, to_dev(evk))
    want0, want1 = o.keyswitch(c0, c1, evk, level)
    assert (got0 == want0).all() and (got1 == want1).all()


def test_keyswitch_c2_decrypts(orc):
    cfg, ctx, o = ctxs(orc, "C2")
    keys, evk = relin_key(o, "C2")
    s2 = o.mul(keys.s_eval, keys.s_eval, list(range(keys.nk)))
    m, c0, c1 = encrypt_under(o, S.rng(5), s2, 29, 20)
    got0, got1 = run_ks(ctx, c0, c1, 29, to_dev(evk))
    dec = o.crt_centered(o.decrypt_coeff(got0, got1, keys.s_eval, 29), 29)
    assert max(abs(a - int(b)) for a, b in zip(dec, m)) <= ks_bound(o, 29, keys.B_e, keys.h)


@pytest.mark.slow
def test_keyswitch_parity_c4(orc):
    """BASELINE.json configs[3] parameters: N=2^17, L=35, dnum=4 (single GPU, unsharded)."""
    cfg, ctx, o = ctxs(orc, "C4")
    g = S.rng(cfg.seed)
    nk = o.nq + o.np
    evk = np.stack([S.uniform_limbs(g, o.primes, o.n) for _ in range(2 * o.dnum)]).reshape(o.dnum, 2, nk, o.n)
    for level in (35, 17):
        c0 = S.uniform_limbs(g, o.q[: level + 1], o.n)
        c1 = S.uniform_limbs(g, o.q[: level + 1], o.n)
        got0, got1 = run_ks(ctx, c0, c1, level, to_dev(evk))
        want0, want1 = o.keyswitch(c0, c1, evk, level)
        assert (got0 == want0).all() and (got1 == want1).all(), level


def test_keyswitch_c0_null_and_determinism(orc):
    cfg, ctx, o = ctxs(orc, "T12")
    keys, evk = relin_key(o, "T12")
    g = S.rng(470)
    level = 6
    c1 = S.uniform_limbs(g, o.q[: level + 1], o.n)
    z = np.zeros_like(c1)
    evk_d = to_dev(evk)
    out0, out1 = empty_dev(c1.shape), empty_dev(c1.shape)
    ws = ctx.workspace(H.OP_KEYSWITCH, level)
    H.keyswitch(ctx, None, to_dev(c1), level, evk_d, out0, out1, ws)
    want0, want1 = o.keyswitch(z, c1, evk, level)
    assert (to_host(out0) == want0).all() and (to_host(out1) == want1).all()
    a0, a1 = run_ks(ctx, z, c1, level, evk_d)
    b0, b1 = run_ks(ctx, z, c1, level, evk_d)
    assert (a0 == b0).all() and (a1 == b1).all() and (a0 == want0).all()


# ------------------------------------------------------------------ hoisted rotations

@pytest.mark.parametrize("name,level,rots", [("T12", 6, [1, 2, 5]), ("C2", 29, [1, 3]),
                                             ("T12", 5, list(range(1, 11))), ("C2", 20, [1, 2, 3, 4, 5, 6, 7, 8, 9])])
def test_rotate_hoisted_parity(orc, name, level, rots):
    cfg, ctx, o = ctxs(orc, name)
    keys = Keys(o, cfg.seed + 11)
    ks = [S.galois_rot(r, cfg.log_n) for r in rots] + [S.GALOIS_CONJ(cfg.log_n)]
    evks = [keys.rot(k) for k in ks]
    g = S.rng(480)
    m, c0, c1 = encrypt_under(o, g, keys.s_eval, level, 20)
    outs0 = [empty_dev(c0.shape) for _ in ks]
    outs1 = [empty_dev(c0.shape) for _ in ks]
    ws = ctx.workspace(H.OP_ROTATE_HOISTED, level, len(ks))
    evk_d = [to_dev(e) for e in evks]
    H.rotate_hoisted(ctx, to_dev(c0), to_dev(c1), level, ks, evk_d, outs0, outs1, ws)
    w0, w1 = o.rotate_hoisted(c0, c1, evks, level, ks)
    for r in range(len(ks)):
        assert (to_host(outs0[r]) == w0[r]).all() and (to_host(outs1[r]) == w1[r]).all(), r


# ------------------------------------------------------------------ error behaviour

def test_error_codes(orc):
    cfg, ctx, o = ctxs(orc, "T12")
    x = empty_dev((2, o.n))
    with pytest.raises(H.HksError) as e:
        H.automorph(ctx, x, 1, 4, x[1:])                     # even Galois element
    assert e.value.status == 7
    with pytest.raises(H.HksError) as e:
        H.automorph(ctx, x, 2, 5, x[1:])                     # overlapping in/out
    assert e.value.status == 1
    with pytest.raises(H.HksError) as e:
        H.ntt_fwd(ctx, x, [0, 99])                           # bad prime index
    assert e.value.status == 1
    with pytest.raises(H.HksError) as e:
        H.modup(ctx, x, 7, x, x)                             # level > L
    assert e.value.status == 1


@pytest.mark.parametrize("name,level", [("T12", 6), ("T12", 3), ("C2", 29), ("C2", 12)])
def test_relinearize_parity(orc, name, level):
    """HMult relinearisation: (d0, d1, d2) -> (d0 + ModDown(acc0), d1 + ModDown(acc1)); bit-exact with the
    oracle's KeySwitch(d0, d2) plus d1, and Dec(out) = d0 + d1 s + d2 s^2 within the bound."""
    cfg, ctx, o = ctxs(orc, name)
    keys, evk = relin_key(o, name)
    g = S.rng(cfg.seed + 31 + level)
    qidx = list(range(level + 1))
    d0, d1, d2 = (S.uniform_limbs(g, o.q[: level + 1], o.n) for _ in range(3))
    out0, out1 = empty_dev(d0.shape), empty_dev(d0.shape)
    ws = ctx.workspace(H.OP_KEYSWITCH, level)
    H.relinearize(ctx, to_dev(d0), to_dev(d1), to_dev(d2), level, to_dev(evk), out0, out1, ws)
    w0, w1 = o.keyswitch(d0, d2, evk, level)
    w1 = o.add(w1, d1, qidx)
    got0, got1 = to_host(out0), to_host(out1)
    assert (got0 == w0).all() and (got1 == w1).all()
    # decryption: out0 + out1 s == d0 + d1 s + d2 s^2 + e_ks
    s_ev = keys.s_eval[: level + 1]
    s2 = o.mul(s_ev, s_ev, qidx)
    ref = o.intt(o.add(o.add(d0, o.mul(d1, s_ev, qidx), qidx), o.mul(d2, s2, qidx), qidx), qidx)
    dec = o.decrypt_coeff(got0, got1, keys.s_eval, level)
    diff = o.crt_centered(o.sub(dec, ref, qidx), level)
    assert max(abs(v) for v in diff) <= ks_bound(o, level, keys.B_e, keys.h)


@pytest.fixture(scope="module")
def experimental_lib():
    """libhks built with -DHKS_EXPERIMENTAL=1 into tools/exp/experimental (built once, ~1 min)."""
    import os, subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = os.path.join(root, "tools", "exp", "experimental", "libhks.so")
    csrc = os.path.join(root, "paper_2507_04775_b200", "csrc")
    newest = max(os.path.getmtime(os.path.join(csrc, f)) for f in os.listdir(csrc))
    if not os.path.exists(out) or os.path.getmtime(out) < newest:
        subprocess.run(["bash", os.path.join(root, "tools", "build_variant.sh"), "experimental", "-DHKS_EXPERIMENTAL=1"],
                       check=True, capture_output=True, timeout=1200)
    return out


@pytest.mark.parametrize("env", [{"HKS_BCONV_FP": "1"}, {"HKS_BCONV_TC": "0"}, {"HKS_BCONV_MMA": "0"},
                                 {"HKS_BCONV_MMA": "0", "HKS_BCONV_KARA": "0"}, {"HKS_NTT_TC": "1"}],
                         ids=["fp64", "imma", "int-kara", "int-plain", "ntt-tensor-cols"])
def test_bconv_alternate_paths_identical(orc, env, experimental_lib):
    """Every base-conversion kernel (tcgen05 default; warp IMMA, integer Karatsuba / plain, FP64-assisted) and
    the tensor-core NTT column pass must produce the same KeySwitch bits as the oracle.  The alternatives are
    measured-and-rejected designs: they exist only in the experimental build
    (-DHKS_EXPERIMENTAL=1, tools/build_variant.sh), selected there by environment switches."""
    import subprocess, sys, os
    env = dict(env, HKS_LIB_PATH=experimental_lib)
    code = ("import sys; sys.path.insert(0, 'tests'); sys.path.insert(0, '.');"
            "import numpy as np, hks_synth as S, oracle; from helpers import *;"
            "from paper_2507_04775_b200 import hks as H;"
            "cfg=S.config('C2'); ctx=H.Context.from_config(cfg,0); o=oracle.Ctx.from_config(cfg); g=S.rng(9);"
            "nk=o.nq+o.np; evk=np.stack([S.uniform_limbs(g,o.primes,o.n) for _ in range(2*o.dnum)]).reshape(o.dnum,2,nk,o.n);"
            "c0=S.uniform_limbs(g,o.q,o.n); c1=S.uniform_limbs(g,o.q,o.n); a,b=empty_dev(c0.shape),empty_dev(c0.shape);"
            "H.keyswitch(ctx,to_dev(c0),to_dev(c1),29,to_dev(evk),a,b,ctx.workspace(H.OP_KEYSWITCH,29));"
            "w0,w1=o.keyswitch(c0,c1,evk,29); assert (to_host(a)==w0).all() and (to_host(b)==w1).all(); print('ok')")
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **env), capture_output=True, text=True, timeout=600,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


@pytest.mark.parametrize("name,level,nct,rots,graph", [("T12", 6, 3, [1, 2, 5], False), ("C2", 29, 2, [1, 3, 8], False),
                                                     ("T12", 5, 2, [1, 2, 3, 4, 5, 6, 7], False),
                                                     ("T12", 4, 3, [1, 3, 5, 7, 9], True)])
def test_rotate_hoisted_batch_parity(orc, name, level, nct, rots, graph):
    """Several ciphertexts sharing rotation keys (C3 shape): each output bit-equal to the hoisted oracle.
    The rotations run round-robin on the caller's stream and the context's side streams (7 rotations:
    several per branch); `graph`: captured into a CUDA graph and replayed."""
    cfg, ctx, o = ctxs(orc, name)
    keys = Keys(o, cfg.seed + 13)
    ks = [S.galois_rot(r, cfg.log_n) for r in rots]
    evks = [keys.rot(k) for k in ks]
    g = S.rng(490)
    cts = [encrypt_under(o, g, keys.s_eval, level, 20)[1:] for _ in range(nct)]
    nr = len(ks)
    outs0 = [empty_dev(cts[0][0].shape) for _ in range(nct * nr)]
    outs1 = [empty_dev(cts[0][0].shape) for _ in range(nct * nr)]
    ws = H.rotate_hoisted_batch_workspace(ctx, nct, level)
    args = (ctx, [to_dev(c[0]) for c in cts], [to_dev(c[1]) for c in cts], level, ks, [to_dev(e) for e in evks],
            outs0, outs1, ws)
    if graph:
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            H.rotate_hoisted_batch(*args, torch.cuda.current_stream().cuda_stream)
        gr.replay()
        torch.cuda.synchronize()
    else:
        H.rotate_hoisted_batch(*args)
    for i, (c0, c1) in enumerate(cts):
        w0, w1 = o.rotate_hoisted(c0, c1, evks, level, ks)
        for r in range(nr):
            assert (to_host(outs0[i * nr + r]) == w0[r]).all() and (to_host(outs1[i * nr + r]) == w1[r]).all(), (i, r)


# ------------------------------------------------------------------ HMult front-end and Rescale (NEXT-1)

def run_hmult(ctx, a0, a1, b0, b1, level, evk_dev):
    out0, out1 = empty_dev(a0.shape), empty_dev(a0.shape)
    ws = ctx.workspace(H.OP_HMULT, level)
    H.hmult(ctx, to_dev(a0), to_dev(a1), to_dev(b0), to_dev(b1), level, evk_dev, out0, out1, ws)
    return to_host(out0), to_host(out1)


@pytest.mark.parametrize("name,levels", [("C1", [2]), ("C1p", [2, 0]), ("T10", [4, 1]), ("T12", [6, 3, 0]),
                                         ("T16s", [5]), ("T17s", [4, 2])])
def test_hmult_parity_small(orc, name, levels):
    """tensor product fused into the first INTT pass (d2) and the ModDown epilogue (d0, d1): bit-exact
    with the oracle's tensor + relinearisation, and decrypts to m1 * m2 within the KS bound."""
    cfg, ctx, o = ctxs(orc, name)
    keys, evk = relin_key(o, name)
    evk_d = to_dev(evk)
    g = S.rng(cfg.seed + 41)
    for level in levels:
        m1, a0, a1 = encrypt_under(o, g, keys.s_eval, level, 12)
        m2, b0, b1 = encrypt_under(o, g, keys.s_eval, level, 12)
        got0, got1 = run_hmult(ctx, a0, a1, b0, b1, level, evk_d)
        want0, want1 = o.hmult(a0, a1, b0, b1, evk, level)
        assert (got0 == want0).all() and (got1 == want1).all(), level


@pytest.mark.parametrize("level", [29, 19, 9, 0])
def test_hmult_parity_c2(orc, level):
    """C2 parameters (N=2^16, L=29, dnum=3) with edge residues, across the digit drops."""
    cfg, ctx, o = ctxs(orc, "C2")
    keys, evk = relin_key(o, "C2")
    g = S.rng(cfg.seed + 200 + level)
    qs = o.q[: level + 1]
    a0, b1 = edge_limbs(qs, o.n, g), edge_limbs(qs, o.n, g)
    a1, b0 = S.uniform_limbs(g, qs, o.n), S.uniform_limbs(g, qs, o.n)
    got0, got1 = run_hmult(ctx, a0, a1, b0, b1, level, to_dev(evk))
    want0, want1 = o.hmult(a0, a1, b0, b1, evk, level)
    assert (got0 == want0).all() and (got1 == want1).all()


@pytest.mark.slow
def test_hmult_parity_c4(orc):
    cfg, ctx, o = ctxs(orc, "C4")
    g = S.rng(cfg.seed + 5)
    nk = o.nq + o.np
    evk = np.stack([S.uniform_limbs(g, o.primes, o.n) for _ in range(2 * o.dnum)]).reshape(o.dnum, 2, nk, o.n)
    level = 35
    a0, a1, b0, b1 = (S.uniform_limbs(g, o.q[: level + 1], o.n) for _ in range(4))
    got0, got1 = run_hmult(ctx, a0, a1, b0, b1, level, to_dev(evk))
    want0, want1 = o.hmult(a0, a1, b0, b1, evk, level)
    assert (got0 == want0).all() and (got1 == want1).all()


def run_rescale(ctx, x, npoly, level):
    out = empty_dev((npoly, level, x.shape[-1]))
    ws = ctx.workspace(H.OP_RESCALE, level, npoly)
    H.rescale(ctx, to_dev(np.ascontiguousarray(x)), npoly, level, out, ws)
    return to_host(out)


@pytest.mark.parametrize("name,levels,npoly", [("C1", [2, 1], 2), ("T10", [4, 1], 1), ("T12", [6, 3, 1], 2),
                                               ("T16s", [5], 3), ("T17s", [4, 1], 2), ("C2", [29, 20, 1], 2),
                                               ("C4", [35], 2)])
def test_rescale_parity(orc, name, levels, npoly):
    """PAPER.md:349 Rescale fusion: SwitchModulo fused into the forward column pass, q_l^-1 (x - .) in
    the row-pass epilogue; bit-exact with the oracle per polynomial."""
    cfg, ctx, o = ctxs(orc, name)
    g = S.rng(cfg.seed + 51)
    for level in levels:
        qs = o.q[: level + 1]
        x = np.stack([edge_limbs(qs, o.n, g) for _ in range(npoly)])
        got = run_rescale(ctx, x, npoly, level)
        for p in range(npoly):
            assert (got[p] == o.rescale(x[p], level)).all(), (level, p)


def test_rescale_many_polys_and_errors(orc):
    """more polynomials than one launch's output table (16), level 0 / overlap rejected."""
    cfg, ctx, o = ctxs(orc, "T12")
    g = S.rng(61)
    level, npoly = 3, 20
    x = np.stack([S.uniform_limbs(g, o.q[: level + 1], o.n) for _ in range(npoly)])
    got = run_rescale(ctx, x, npoly, level)
    for p in (0, 7, 15, 16, 19):
        assert (got[p] == o.rescale(x[p], level)).all(), p
    xd = to_dev(x[0])
    ws = ctx.workspace(H.OP_RESCALE, 1, 1)
    with pytest.raises(H.HksError) as e:
        H.rescale(ctx, xd, 1, 0, empty_dev((1, o.n)), ws)            # level 0
    assert e.value.status == 1
    with pytest.raises(H.HksError) as e:
        H.rescale(ctx, xd, 1, level, xd, ws)                         # out overlaps x
    assert e.value.status == 1


def test_hmult_rejects_aliasing(orc):
    cfg, ctx, o = ctxs(orc, "T12")
    keys, evk = relin_key(o, "T12")
    level = 2
    a = to_dev(S.uniform_limbs(S.rng(1), o.q[: level + 1], o.n))
    out1 = empty_dev(a.shape)
    ws = ctx.workspace(H.OP_HMULT, level)
    with pytest.raises(H.HksError) as e:
        H.hmult(ctx, a, a, a, a, level, to_dev(evk), a, out1, ws)    # out0 aliases an input
    assert e.value.status == 1


# ------------------------------------------------------------------ BSGS linear transform (NEXT-2)

@pytest.mark.parametrize("name,level,nterm", [("T12", 6, 5), ("T12", 3, 21), ("C2", 29, 8)])
def test_pt_weighted_sum_parity(orc, name, level, nterm):
    """fused weighted sum, incl. > 16 terms (second pass accumulates into the outputs)."""
    cfg, ctx, o = ctxs(orc, name)
    g = S.rng(cfg.seed + 71 + nterm)
    qs = o.q[: level + 1]
    w = [edge_limbs(qs, o.n, g) for _ in range(nterm)]
    x0 = [S.uniform_limbs(g, qs, o.n) for _ in range(nterm)]
    x1 = [edge_limbs(qs, o.n, g) for _ in range(nterm)]
    out0, out1 = empty_dev(x0[0].shape), empty_dev(x0[0].shape)
    H.pt_weighted_sum(ctx, [to_dev(v) for v in w], [to_dev(v) for v in x0], [to_dev(v) for v in x1], level, out0, out1)
    w0, w1 = o.pt_wsum(w, x0, x1, level)
    assert (to_host(out0) == w0).all() and (to_host(out1) == w1).all()


@pytest.mark.parametrize("name,level,n1,n2,graph", [("T12", 6, 3, 3, False), ("T12", 4, 4, 1, False),
                                                    ("T12", 5, 1, 3, False), ("T12", 2, 1, 1, False),
                                                    ("T12", 6, 2, 8, False), ("T12", 3, 3, 5, True),
                                                    ("T12", 6, 2, 8, True), ("C2", 29, 4, 4, False)])
def test_linear_transform_parity(orc, name, level, n1, n2, graph):
    """BSGS: hoisted baby rotations, fused weighted sums, one rotation per giant step; bit-exact.  n2 > 2:
    the giant steps run round-robin on the caller's stream and the context's side streams (n2 = 8: every
    branch takes several steps); `graph`: the call captured into a CUDA graph (fork / join inside the
    capture) and replayed."""
    cfg, ctx, o = ctxs(orc, name)
    keys = Keys(o, cfg.seed + 81)
    g = S.rng(cfg.seed + 82)
    bgal = [S.galois_rot(j, cfg.log_n) for j in range(1, n1)]
    ggal = [S.galois_rot(i * n1, cfg.log_n) for i in range(1, n2)]
    bk = [keys.rot(k) for k in bgal]
    gk = [keys.rot(k) for k in ggal]
    qs = o.q[: level + 1]
    c0, c1 = S.uniform_limbs(g, qs, o.n), edge_limbs(qs, o.n, g)
    pts = [S.uniform_limbs(g, qs, o.n) for _ in range(n1 * n2)]
    out0, out1 = empty_dev(c0.shape), empty_dev(c0.shape)
    ws = H.linear_transform_workspace(ctx, level, n1)
    args = (ctx, to_dev(c0), to_dev(c1), level, n1, n2, bgal, [to_dev(k) for k in bk], ggal,
            [to_dev(k) for k in gk], [to_dev(p) for p in pts], out0, out1, ws)
    if graph:
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            H.linear_transform(*args, torch.cuda.current_stream().cuda_stream)
        gr.replay()
        torch.cuda.synchronize()
    else:
        H.linear_transform(*args)
    w0, w1 = o.lintrans(c0, c1, level, n1, n2, bgal, bk, ggal, gk, pts)
    assert (to_host(out0) == w0).all() and (to_host(out1) == w1).all()


def test_keyswitch_batch_shared_key_parity(orc):
    """a batch of ciphertexts relinearised with one key = hks_rotate_hoisted_batch with Galois 1 (the
    identity): each output is bit-exactly the oracle's single-ciphertext KeySwitch."""
    cfg, ctx, o = ctxs(orc, "C2")
    keys, evk = relin_key(o, "C2")
    level, nct = 29, 3
    g = S.rng(91)
    c0s = [S.uniform_limbs(g, o.q[: level + 1], o.n) for _ in range(nct)]
    c1s = [edge_limbs(o.q[: level + 1], o.n, g) for _ in range(nct)]
    outs0 = [empty_dev(c0s[0].shape) for _ in range(nct)]
    outs1 = [empty_dev(c0s[0].shape) for _ in range(nct)]
    ws = H.rotate_hoisted_batch_workspace(ctx, nct, level)
    H.rotate_hoisted_batch(ctx, [to_dev(c) for c in c0s], [to_dev(c) for c in c1s], level, [1], [to_dev(evk)],
                           outs0, outs1, ws)
    for i in range(nct):
        w0, w1 = o.keyswitch(c0s[i], c1s[i], evk, level)
        assert (to_host(outs0[i]) == w0).all() and (to_host(outs1[i]) == w1).all(), i


def test_keyswitch_after_cross_stream_copy(orc):
    """Programmatic dependent launch must not let a KeySwitch start before a cross-stream dependency
    (an H2D copy ordered by an event) completes: the e2e pipeline and any caller rely on it."""
    import torch
    cfg, ctx, o = ctxs(orc, "C2")
    dev = "cuda:0"
    g = torch.Generator(device=dev)
    g.manual_seed(77)
    n, level = cfg.n, 29
    prim = list(cfg.q) + list(cfg.p)

    def limbs(pr):
        return torch.stack([torch.randint(0, int(p), (n,), generator=g, device=dev, dtype=torch.int64) for p in pr])

    evk = torch.stack([limbs(prim) for _ in range(2 * cfg.dnum)]).reshape(cfg.dnum, 2, len(prim), n)
    cts = [(limbs(cfg.q), limbs(cfg.q)) for _ in range(3)]
    ws = ctx.workspace(H.OP_KEYSWITCH, level)
    refs = []
    for c0, c1 in cts:
        r0, r1 = torch.empty_like(c0), torch.empty_like(c1)
        H.keyswitch(ctx, c0, c1, level, evk, r0, r1, ws)
        refs.append((r0, r1))
    host = [(c0.cpu().pin_memory(), c1.cpu().pin_memory()) for c0, c1 in cts]
    d0, d1 = torch.empty_like(cts[0][0]), torch.empty_like(cts[0][1])
    s_cmp, s_cpy = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    outs = [(torch.empty_like(d0), torch.empty_like(d1)) for _ in range(9)]
    e_done, e_in = torch.cuda.Event(), torch.cuda.Event()
    torch.cuda.synchronize()
    for i in range(9):
        k = i % 3
        with torch.cuda.stream(s_cpy):
            s_cpy.wait_event(e_done)                # previous KeySwitch has read d0, d1
            d0.copy_(host[k][0], non_blocking=True)
            d1.copy_(host[k][1], non_blocking=True)
            e_in.record(s_cpy)
        s_cmp.wait_event(e_in)
        H.keyswitch(ctx, d0, d1, level, evk, outs[i][0], outs[i][1], ws, s_cmp.cuda_stream)
        e_done.record(s_cmp)
    torch.cuda.synchronize()
    for i in range(9):
        assert torch.equal(outs[i][0], refs[i % 3][0]) and torch.equal(outs[i][1], refs[i % 3][1]), i


@pytest.mark.parametrize("name,level,nstream", [("C2", 29, 3), ("C1", 2, 8)])
def test_concurrent_keyswitches_on_streams(orc, name, level, nstream):
    """bench.py's batch step: `nstream` KeySwitches of distinct ciphertexts, each on its own stream with its
    own workspace, forked from and joined to the current stream (directly and as one captured CUDA graph):
    every output equals the oracle's."""
    import torch
    cfg, ctx, o = ctxs(orc, name)
    g = S.rng(cfg.seed + 31)
    nk = o.nq + o.np
    evk = np.stack([S.uniform_limbs(g, o.primes, o.n) for _ in range(2 * o.dnum)]).reshape(o.dnum, 2, nk, o.n)
    evk_d = to_dev(evk)
    cts = [(S.uniform_limbs(g, o.q[: level + 1], o.n), S.uniform_limbs(g, o.q[: level + 1], o.n))
           for _ in range(nstream)]
    want = [o.keyswitch(c0, c1, evk, level) for c0, c1 in cts]
    dcts = [(to_dev(c0), to_dev(c1)) for c0, c1 in cts]
    outs = [(torch.empty_like(a), torch.empty_like(b)) for a, b in dcts]
    wss = [ctx.workspace(H.OP_KEYSWITCH, level) for _ in range(nstream)]
    sts = [torch.cuda.Stream() for _ in range(nstream)]

    def batch():
        cur = torch.cuda.current_stream()
        for st in sts:
            st.wait_stream(cur)
        for j, st in enumerate(sts):
            H.keyswitch(ctx, dcts[j][0], dcts[j][1], level, evk_d, outs[j][0], outs[j][1], wss[j], st.cuda_stream)
        for st in sts:
            cur.wait_stream(st)

    def check():
        torch.cuda.synchronize()
        for j in range(nstream):
            assert (to_host(outs[j][0]) == want[j][0]).all() and (to_host(outs[j][1]) == want[j][1]).all(), j
            outs[j][0].zero_()
            outs[j][1].zero_()

    batch()
    check()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        batch()
    graph.replay()
    check()


def test_linear_transform_two_host_threads(orc):
    """Two host threads run BSGS transforms on one context concurrently (own streams and workspaces): the
    context's side streams are shared under its mutex, and both results equal the oracle's."""
    import threading
    cfg, ctx, o = ctxs(orc, "T12")
    keys = Keys(o, cfg.seed + 91)
    level, n1, n2 = 5, 2, 6
    bgal = [S.galois_rot(j, cfg.log_n) for j in range(1, n1)]
    ggal = [S.galois_rot(i * n1, cfg.log_n) for i in range(1, n2)]
    bk, gk = [keys.rot(k) for k in bgal], [keys.rot(k) for k in ggal]
    bkd, gkd = [to_dev(k) for k in bk], [to_dev(k) for k in gk]
    qs = o.q[: level + 1]
    jobs = []
    for t in range(2):
        g = S.rng(cfg.seed + 92 + t)
        c0, c1 = S.uniform_limbs(g, qs, o.n), S.uniform_limbs(g, qs, o.n)
        pts = [S.uniform_limbs(g, qs, o.n) for _ in range(n1 * n2)]
        jobs.append(dict(c0=c0, c1=c1, pts=pts, d0=to_dev(c0), d1=to_dev(c1), dp=[to_dev(p) for p in pts],
                         out0=empty_dev(c0.shape), out1=empty_dev(c0.shape),
                         ws=H.linear_transform_workspace(ctx, level, n1), st=torch.cuda.Stream()))
    torch.cuda.synchronize()
    errs = []

    def work(j):
        try:
            for _ in range(5):
                H.linear_transform(ctx, j["d0"], j["d1"], level, n1, n2, bgal, bkd, ggal, gkd, j["dp"], j["out0"],
                                   j["out1"], j["ws"], j["st"].cuda_stream)
        except Exception as e:   # pragma: no cover - reported below
            errs.append(e)

    th = [threading.Thread(target=work, args=(j,)) for j in jobs]
    for t in th:
        t.start()
    for t in th:
        t.join()
    torch.cuda.synchronize()
    assert not errs, errs
    for j in jobs:
        w0, w1 = o.lintrans(j["c0"], j["c1"], level, n1, n2, bgal, bk, ggal, gk, j["pts"])
        assert (to_host(j["out0"]) == w0).all() and (to_host(j["out1"]) == w1).all()


def test_hoisted_and_bsgs_under_profiling(orc):
    """With per-kernel profiling on, the branch-parallel calls keep every branch on the caller's stream
    (workspaces sized for the concurrent layout): results still equal the oracle."""
    cfg, ctx, o = ctxs(orc, "T12")
    keys = Keys(o, cfg.seed + 95)
    level, rots = 5, [1, 2, 3, 4, 5, 6, 7]
    ks = [S.galois_rot(r, cfg.log_n) for r in rots]
    evks = [keys.rot(k) for k in ks]
    g = S.rng(496)
    c0, c1 = S.uniform_limbs(g, o.q[: level + 1], o.n), S.uniform_limbs(g, o.q[: level + 1], o.n)
    outs0 = [empty_dev(c0.shape) for _ in ks]
    outs1 = [empty_dev(c0.shape) for _ in ks]
    ws = ctx.workspace(H.OP_ROTATE_HOISTED, level, len(ks))
    H.prof_enable(True)
    try:
        H.rotate_hoisted(ctx, to_dev(c0), to_dev(c1), level, ks, [to_dev(e) for e in evks], outs0, outs1, ws)
        torch.cuda.synchronize()
    finally:
        H.prof_enable(False)
        H.prof_read()
    w0, w1 = o.rotate_hoisted(c0, c1, evks, level, ks)
    for r in range(len(ks)):
        assert (to_host(outs0[r]) == w0[r]).all() and (to_host(outs1[r]) == w1[r]).all(), r


# ------------------------------------------------------------------ prepared keys (hks_evk_prepare)

@pytest.mark.parametrize("name,levels", [("C2", [29, 19, 9, 0]), ("T12", [6, 3, 0]), ("C1p", [2, 0]), ("T16s", [5, 1])])
def test_prepared_key_keyswitch_parity(orc, name, levels):
    """include/hks.h hks_evk_prepare (optional): a key with P^-1 on its Q limbs and the
    P^-1-folded ModDown matrix give the oracle's KeySwitch bit for bit -- the oracle is unchanged, so this is
    the same pin as every KeySwitch parity test (fused path at beta <= 4, and the small configs)."""
    cfg, ctx, o = ctxs(orc, name)
    keys, evk = relin_key(o, name)
    pk = H.evk_prepare(ctx, to_dev(evk), out=empty_dev(evk.shape))
    prep = to_host(pk.tensor)
    assert not (prep == evk).all()                         # the Q limbs did change
    assert (prep[:, :, o.nq:] == evk[:, :, o.nq:]).all()   # the P limbs did not
    g = S.rng(cfg.seed + 300)
    for level in levels:
        c0 = S.uniform_limbs(g, o.q[: level + 1], o.n)
        c1 = edge_limbs(o.q[: level + 1], o.n, g)
        got0, got1 = run_ks(ctx, c0, c1, level, pk)
        want0, want1 = o.keyswitch(c0, c1, evk, level)
        assert (got0 == want0).all() and (got1 == want1).all(), level


def test_prepared_key_hmult_rotations_and_errors(orc):
    """The prepared key through HMult (tensor terms after the ModDown core), hoisted rotations (batched
    ModDowns with per-rotation outputs) and the in-place form; the step-level key product and a second
    preparation refuse it."""
    cfg, ctx, o = ctxs(orc, "T12")
    keys, evk = relin_key(o, "T12")
    level = 5
    g = S.rng(cfg.seed + 310)
    qs = o.q[: level + 1]
    a0, a1, b0, b1 = (S.uniform_limbs(g, qs, o.n) for _ in range(4))
    pk = H.evk_prepare(ctx, to_dev(evk))                   # in place
    got0, got1 = run_hmult(ctx, a0, a1, b0, b1, level, pk)
    want0, want1 = o.hmult(a0, a1, b0, b1, evk, level)
    assert (got0 == want0).all() and (got1 == want1).all()
    rk = Keys(o, cfg.seed + 11)
    ks = [S.galois_rot(r, cfg.log_n) for r in (1, 2, 5)]
    evks = [rk.rot(k) for k in ks]
    pks = [H.evk_prepare(ctx, to_dev(e)) for e in evks]
    m, c0, c1 = encrypt_under(o, g, rk.s_eval, level, 20)
    outs0 = [empty_dev(c0.shape) for _ in ks]
    outs1 = [empty_dev(c0.shape) for _ in ks]
    H.rotate_hoisted(ctx, to_dev(c0), to_dev(c1), level, ks, pks, outs0, outs1,
                     ctx.workspace(H.OP_ROTATE_HOISTED, level, len(ks)))
    w0, w1 = o.rotate_hoisted(c0, c1, evks, level, ks)
    for r in range(len(ks)):
        assert (to_host(outs0[r]) == w0[r]).all() and (to_host(outs1[r]) == w1[r]).all(), r
    with pytest.raises(ValueError):
        H.evk_digits(ctx, [pks[0], to_dev(evks[1])])
    ext = empty_dev((o.dnum, level + 1 + o.np, o.n))
    acc = empty_dev((2, level + 1 + o.np, o.n))
    with pytest.raises(H.HksError) as ei:
        H.ksk_inner_product(ctx, ext, pk, level, 1, acc)
    assert ei.value.status == 1
    with pytest.raises(H.HksError) as ei:
        H.evk_prepare(ctx, pk)
    assert ei.value.status == 1
