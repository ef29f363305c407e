"""Level and limb-batch sweeps (SURVEY.md 8(d) "level-sweep curve", 8(f) NEXT-4; PAPER.md:499-524,
figs 7-8: throughput vs level and vs limb batch). Run on the GPU box:

  python tools/sweep.py --out gpurun_out/sweep.json      # then, here:
  python tools/sweep.py --render gpurun_out/sweep.json --name r1   -> profiles/sweep_<name>.md

Timing follows bench.py: warm-up, CUDA events on the launching stream, inputs rotated over sets
larger than L2 (KS) or 4 buffers (NTT).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def time_it(torch, stream, fn, it, warm=5):
    for i in range(warm):
        fn(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(it):
        fn(i)
    e1.record(stream)
    e1.synchronize()
    return e0.elapsed_time(e1) / it


def run(out):
    import torch
    import hks_synth as S
    import bench
    from paper_2507_04775_b200 import hks as H
    torch.cuda.set_device(0)
    dev = "cuda:0"
    stream = torch.cuda.current_stream()
    sid = stream.cuda_stream
    res = {"levels": {}, "ntt": {}}

    # ---- C2 level sweep: one relinearisation KS per step at every level 29..0
    cfg = S.config("C2")
    ctx = H.Context.from_config(cfg, 0)
    for level in range(cfg.L, -1, -1):
        wl = bench.KSWorkload(H, ctx, cfg, level, 4, dev, 77, sid)
        ms = time_it(torch, stream, wl.step, 100)
        res["levels"][level] = {"ms": ms, "ks_per_s": 1e3 / ms, "beta": cfg.beta(level)}
        del wl
        torch.cuda.empty_cache()
    del ctx

    # ---- NTT limb-batch sweep at N = 2^12 / 2^16 / 2^17, fwd and inv
    for name in ("C1", "C2", "C4"):
        cfg = S.config(name)
        ctx = H.Context.from_config(cfg, 0)
        nprime = len(cfg.q) + len(cfg.p)
        for nl in (1, 2, 4, 8, 16, 30, 45, 60, 90, 120, 150):
            idx = [i % nprime for i in range(nl)]
            bufs = [torch.randint(0, int(min(cfg.q + cfg.p)), (nl, cfg.n), device=dev, dtype=torch.int64)
                    for _ in range(4)]
            for kind, fn in (("fwd", H.ntt_fwd), ("inv", H.ntt_inv)):
                ms = time_it(torch, stream, lambda i: fn(ctx, bufs[i % 4], idx, sid), 50)
                res["ntt"].setdefault(str(cfg.n), {}).setdefault(kind, {})[nl] = {
                    "us": ms * 1e3, "limbs_per_s": nl / (ms * 1e-3),
                    "hbm_gbs": 2 * nl * cfg.n * 8 / (ms * 1e-3) / 1e9}
            del bufs
        del ctx
        torch.cuda.empty_cache()
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res)[:2000])


def render(path, name):
    r = json.load(open(path))
    md = [f"# Sweeps: {name}", "",
          "`python tools/sweep.py` on 1x B200 (CUDA events, warm-up 5, inputs rotated). "
          "SURVEY.md 8(d) level sweep; 8(f) NEXT-4 (PAPER.md:499-524).", "",
          "## C2 KeySwitch vs level (N=2^16, L=29, K=10, dnum=3)", "",
          "| level | beta | µs/KS | KS/s |", "|---|---|---|---|"]
    for lv, v in sorted(r["levels"].items(), key=lambda kv: -int(kv[0])):
        md.append(f"| {lv} | {v['beta']} | {v['ms'] * 1e3:.1f} | {v['ks_per_s']:.0f} |")
    for n, kinds in r["ntt"].items():
        md += ["", f"## NTT limb batch at N={n}", "",
               "| limbs | fwd µs | fwd M limbs/s | fwd GB/s | inv µs | inv M limbs/s | inv GB/s |",
               "|---|---|---|---|---|---|---|"]
        for nl in kinds["fwd"]:
            f, i = kinds["fwd"][nl], kinds["inv"][nl]
            md.append(f"| {nl} | {f['us']:.1f} | {f['limbs_per_s'] / 1e6:.2f} | {f['hbm_gbs']:.0f} | "
                      f"{i['us']:.1f} | {i['limbs_per_s'] / 1e6:.2f} | {i['hbm_gbs']:.0f} |")
    p = os.path.join(ROOT, "profiles", f"sweep_{name}.md")
    with open(p, "w") as f:
        f.write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/sweep.json")
    ap.add_argument("--render")
    ap.add_argument("--name", default="r1")
    a = ap.parse_args()
    if a.render:
        render(a.render, a.name)
    else:
        run(a.out)
