"""Diagnostic: batched NTT time with the batch L2-resident (one 45 MiB buffer reused) vs HBM-resident
(4 rotating buffers, 180 MiB).  Equal times => the NTT passes are not memory-latency/bandwidth bound."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import hks_synth as S
from paper_2507_04775_b200 import hks as H

cfg = S.config("C2")
ctx = H.Context.from_config(cfg, 0)
nl = 90
idx = [i % 40 for i in range(nl)]
res = {}
for nbuf in (1, 4):
    bufs = [torch.randint(0, int(cfg.p[-1]), (nl, cfg.n), device="cuda:0", dtype=torch.int64) for _ in range(nbuf)]
    for kind, fn in (("fwd", H.ntt_fwd), ("inv", H.ntt_inv)):
        for i in range(5):
            fn(ctx, bufs[i % nbuf], idx)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        H.prof_enable(True)
        e0.record()
        for i in range(50):
            fn(ctx, bufs[i % nbuf], idx)
        e1.record()
        e1.synchronize()
        prof = H.prof_read()
        H.prof_enable(False)
        res[f"{kind}_bufs{nbuf}_us_per_batch"] = e0.elapsed_time(e1) / 50 * 1e3
        res[f"{kind}_bufs{nbuf}_passes_us"] = {k: round(v[1] / v[0] * 1e3, 2) for k, v in prof.items()}
print(json.dumps(res, indent=1))
