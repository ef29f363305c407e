"""Small end-to-end exercise of every product kernel for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck), checked against the oracle.  Usage (GPU box):
  compute-sanitizer --tool racecheck python tools/sanitize_run.py C1
Configs: C1 (N = 2^12, integer-pipe base conversions) and T16s (N = 2^16, 60-bit primes: the tcgen05
base-conversion kernel, the fused row pass + key product, every NTT shape of the KeySwitch)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import hks_synth as S  # noqa: E402
import oracle  # noqa: E402
from helpers import empty_dev, to_dev, to_host  # noqa: E402
from paper_2507_04775_b200 import hks as H  # noqa: E402


def main(name):
    cfg = S.config(name)
    ctx = H.Context.from_config(cfg, 0)
    o = oracle.Ctx.from_config(cfg)
    g = S.rng(cfg.seed + 5)
    L = cfg.L
    nk = len(cfg.q) + len(cfg.p)
    evk = np.stack([S.uniform_limbs(g, o.primes, o.n) for _ in range(2 * cfg.dnum)]).reshape(cfg.dnum, 2, nk, o.n)
    ek = to_dev(evk)
    c0, c1, b0, b1 = (S.uniform_limbs(g, o.q, o.n) for _ in range(4))
    ok = []
    # NTT round trip over every prime
    idx = list(range(nk))
    x = S.uniform_limbs(g, o.primes, o.n)
    d = to_dev(x)
    H.ntt_fwd(ctx, d, idx)
    ok.append((to_host(d) == o.ntt(x, idx)).all())
    H.ntt_inv(ctx, d, idx)
    ok.append((to_host(d) == x).all())
    for level in sorted({L, max(0, L - 2)}):
        l1 = level + 1
        a0, a1 = empty_dev((l1, o.n)), empty_dev((l1, o.n))
        H.keyswitch(ctx, to_dev(c0[:l1]), to_dev(c1[:l1]), level, ek, a0, a1, ctx.workspace(H.OP_KEYSWITCH, level))
        w0, w1 = o.keyswitch(c0[:l1], c1[:l1], evk, level)
        ok.append((to_host(a0) == w0).all() and (to_host(a1) == w1).all())
        H.hmult(ctx, to_dev(c0[:l1]), to_dev(c1[:l1]), to_dev(b0[:l1]), to_dev(b1[:l1]), level, ek, a0, a1,
                ctx.workspace(H.OP_HMULT, level))
        w0, w1 = o.hmult(c0[:l1], c1[:l1], b0[:l1], b1[:l1], evk, level)
        ok.append((to_host(a0) == w0).all() and (to_host(a1) == w1).all())
        if level >= 1:
            rs = empty_dev((2, level, o.n))
            H.rescale(ctx, torch.stack([a0, a1]), 2, level, rs, ctx.workspace(H.OP_RESCALE, level, 2))
            got = to_host(rs)
            ok.append((got[0] == o.rescale(w0, level)).all() and (got[1] == o.rescale(w1, level)).all())
        gal = [S.galois_rot(1, cfg.log_n), S.galois_rot(3, cfg.log_n)]
        outs0 = [empty_dev((l1, o.n)) for _ in gal]
        outs1 = [empty_dev((l1, o.n)) for _ in gal]
        H.rotate_hoisted(ctx, to_dev(c0[:l1]), to_dev(c1[:l1]), level, gal, [ek, ek], outs0, outs1,
                         ctx.workspace(H.OP_ROTATE_HOISTED, level, len(gal)))
        w0s, w1s = o.rotate_hoisted(c0[:l1], c1[:l1], [evk, evk], level, gal)
        ok.append(all((to_host(outs0[k]) == w0s[k]).all() and (to_host(outs1[k]) == w1s[k]).all()
                      for k in range(len(gal))))
    src, dst = list(range(min(3, len(cfg.q)))), list(range(min(3, len(cfg.q)), nk))
    xs = S.uniform_limbs(g, [o.primes[i] for i in src], o.n)
    out = empty_dev((len(dst), o.n))
    H.bconv(ctx, to_dev(xs), src, dst, out)
    ok.append((to_host(out) == o.bconv(xs, src, dst)).all())
    torch.cuda.synchronize()
    print(name, "checks:", len(ok), "all bit-exact" if all(ok) else f"MISMATCH {ok}")
    return all(ok)


if __name__ == "__main__":
    sys.exit(0 if all(main(n) for n in (sys.argv[1:] or ["C1", "T16s"])) else 1)
