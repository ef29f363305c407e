"""Debug helper: localise a ModDown mismatch (which limbs / positions differ)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import hks_synth as S
import oracle
from paper_2507_04775_b200 import hks as H
from helpers import to_dev, to_host, empty_dev

for name, level in (("T12", 6), ("T12", 1), ("C2", 29), ("T10", 4)):
    cfg = S.config(name)
    ctx = H.Context.from_config(cfg, 0)
    o = oracle.Ctx.from_config(cfg)
    g = S.rng(460 + level)
    eidx = o.ext_primes(level)
    acc = S.uniform_limbs(g, [o.primes[i] for i in eidx], o.n)
    out = empty_dev((level + 1, o.n))
    ws = ctx.workspace(H.OP_MODDOWN, level)
    H.moddown(ctx, to_dev(acc), level, out, ws)
    got = to_host(out)
    want = o.moddown(acc, level)
    bad = got != want
    print(name, level, "mismatch frac", bad.mean(), "per limb", bad.mean(axis=1).round(3).tolist())
    if bad.any():
        l, x = np.argwhere(bad)[0]
        q = o.q[l]
        print("  first", l, x, int(got[l, x]), int(want[l, x]), "q", q, "got>=q", int(got[l, x]) >= q,
              "diff mod q", (int(got[l, x]) - int(want[l, x])) % q)
