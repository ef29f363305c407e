#!/usr/bin/env python
"""bench.py -- hybrid key switching on B200 (BASELINE.json metric), one JSON line on rank 0.

Default workload (BASELINE.json configs[1], `C2`): one relinearisation KeySwitch of one ciphertext at
N=2^16, L=29 (30 Q limbs), K=10 special primes, dnum=3, 60-bit primes, level 29.  A step = one
KeySwitch (all of SURVEY.md §8(a): INTT, ModUp BConv, NTT, key inner product, ModDown) per ciphertext of
a batch of `--streams` independent ciphertexts, each on its own CUDA stream with its own workspace (the
throughput-with-batch setting of the paper's throughput figures; `--streams 1` = one KeySwitch at a time).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl hks|reference] [--config C2|C1|C4]
  torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU, ciphertexts sharded: weak scaling)

Timing: W untimed steps, then K steps between barrier + synchronize, CUDA events on the launch
stream, max over ranks.  L2: every step uses the next of `--sets` distinct (ciphertext, key) sets
(total > 4x the device's L2, read from cudaDevAttrL2CacheSize), so nothing is L2-resident from the
previous step.
Inputs are seeded synthetic residues (timing is data-independent; bit-exactness with real keys is
the job of tests/test_gpu_parity.py).  `--impl reference` times the CPU oracle (oracle/) instead.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import hks_synth as S  # noqa: E402

METRIC = "KeySwitch ops/s at N=2^16,L=29,dnum=3; NTT limbs/s; % HBM peak"
HBM_FALLBACK_GBS = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="hks", choices=["hks", "reference"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--level", type=int, default=None)
    ap.add_argument("--sets", type=int, default=5)
    ap.add_argument("--streams", type=int, default=0,
                    help="C1/C2/C4: ciphertexts KeySwitched concurrently per step, one CUDA stream each "
                         "(0 = the measured best per config: C1 8, C2 3, C4 2)")
    ap.add_argument("--key", choices=("prepared", "plain"), default="prepared",
                    help="C1/C2/C4: keys prepared once at load time with hks_evk_prepare (P^-1 on the Q limbs, "
                         "outside the timed region; bit-identical outputs) or used as generated")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--quick", action="store_true", help="skip e2e / NTT / profile legs (for ncu runs)")
    ap.add_argument("--no-graph", action="store_true",
                    help="time direct C-ABI calls instead of CUDA-graph replays of the same calls")
    ap.add_argument("--dump", default=None,
                    help="directory: after the timed region every rank saves one step's inputs and outputs (.npy) "
                         "for an offline oracle check (tests/test_multirank.py)")
    ap.add_argument("--shard", default="auto", choices=["auto", "none", "nccl", "pipe", "a2a", "peer"],
                    help="C4 limb sharding: nccl = two NCCL all-gathers per KeySwitch; pipe = the first exchange as "
                         "per-digit broadcasts overlapped with the conversions; a2a = coefficient-sharded "
                         "conversions with four all-to-alls; peer = the exchanges fused into the "
                         "base conversions over NVLink symmetric memory; none = one KeySwitch per GPU; auto = nccl "
                         "for C4 under torchrun, else none")
    return ap.parse_args()


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return HBM_FALLBACK_GBS, "fallback (B200_PROFILING.md)"


def tensor_peak():
    """Dense u8 tensor-core ops/s: the measured bf16 burst rate (MEASURED_PEAKS.json) x 2, the nominal int8 /
    bf16 ratio of B200_PROFILING.md; fallback: the nominal 4.5 POPS."""
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return 2e12 * float(d["bf16_tflops"]), "measured bf16 x 2 (MEASURED_PEAKS.json bf16_tflops)"
    return 4.5e15, "nominal int8 dense"


L2_BYTES = 126 * 1024 * 1024   # replaced in main() by the device's cudaDevAttrL2CacheSize


def l2_str():
    return f"{L2_BYTES / 2**20:.0f} MiB L2"


def mul_peak():
    """Peak 32x32->64-bit integer multiplies/s (IMAD.WIDE / IMAD.HI, half-rate FMA-pipe ops), measured
    by tools/int_probe.cu on this pool's B200 (profiles/int_probe.json, imad_hi); fallback: the
    nominal 32 per SM per clock x 148 SMs x 1.965 GHz."""
    path = os.path.join(ROOT, "profiles", "int_probe.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return float(d["imad_hi"]["ops_per_s"]), "measured (profiles/int_probe.json imad_hi)"
    return 32 * 148 * 1.965e9, "nominal (32/clk/SM x 148 x 1.965 GHz)"


def workload_desc(cfg, level):
    base = f"N=2^{cfg.log_n}, L={cfg.L}, K={cfg.K}, dnum={cfg.dnum}"
    if cfg.name == "C3":
        return (f"C3: 8 ciphertexts x 8 hoisted rotation KeySwitches (r=1..8, Galois 5^r), {base}, level={level}, "
                f"keys replicated, ciphertexts sharded over ranks")
    if cfg.name == "C5":
        return (f"C5: BOOT_SHAPE v2 (DESIGN.md reading 14): CtS 3x(BSGS linear transform n1=n2=8: 7 hoisted baby "
                f"+ 7 giant rotations, 64 diagonals; Rescale) at l=29..27, conjugation at 26, EvalMod stand-in "
                f"12x(HMult + Rescale) at l=26..15, StC 3x(BSGS + Rescale) at l=14..12 = 97 KeySwitches, {base}")
    return f"{cfg.name}: one relinearisation KeySwitch per ciphertext, {base}, level={level}, primes<2^{cfg.bits}"


# ---------------------------------------------------------------------------------------------- clocks
class ClockSampler:
    """NVML sampling of SM clock and clock-event reasons DURING the timed region."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, dev_index: int):
        self.ok = False
        self.samples, self.reasons = [], 0
        try:
            import pynvml
            import torch
            pynvml.nvmlInit()
            self.nv = pynvml
            h = None
            try:
                uuid = str(torch.cuda.get_device_properties(dev_index).uuid)
                h = pynvml.nvmlDeviceGetHandleByUUID(uuid if uuid.startswith("GPU-") else "GPU-" + uuid)
            except Exception:
                h = pynvml.nvmlDeviceGetHandleByIndex(dev_index)
            self.h = h
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)

    def _loop(self):
        nv = self.nv
        get_r = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or nv.nvmlDeviceGetCurrentClocksThrottleReasons
        while not self.stop:
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.reasons |= int(get_r(self.h))
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.ok:
            self.stop = False
            self.t = threading.Thread(target=self._loop, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self.stop = True
            self.t.join()

    def summary(self):
        if not self.ok:
            return {"error": getattr(self, "err", "nvml unavailable")}
        s = sorted(self.samples)
        med = s[len(s) // 2] if s else None
        reasons = [v for k, v in self.REASONS.items() if self.reasons & k and k != 0x1]
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(s)}


# ---------------------------------------------------------------------------------------------- inputs
def make_sets(cfg, level, nsets, dev, seed):
    """Seeded uniform residues per limb, generated on the device (torch Philox, seed per rank)."""
    import torch
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    n = cfg.n
    primes = list(cfg.q) + list(cfg.p)
    nk = len(primes)

    def limbs(pr):
        t = torch.empty((len(pr), n), dtype=torch.int64, device=dev)
        for i, q in enumerate(pr):
            t[i] = torch.randint(0, int(q), (n,), generator=g, device=dev, dtype=torch.int64)
        return t

    sets = []
    for _ in range(nsets):
        c0 = limbs(cfg.q[: level + 1])
        c1 = limbs(cfg.q[: level + 1])
        evk = torch.stack([limbs(primes) for _ in range(2 * cfg.dnum)]).reshape(cfg.dnum, 2, nk, n)
        sets.append({"c0": c0, "c1": c1, "evk": evk,
                     "out0": torch.empty_like(c0), "out1": torch.empty_like(c1)})
    return sets


# ---------------------------------------------------------------------------------------------- cpu
def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def oracle_ks_timer(cfg, level, seed):
    import numpy as np
    import oracle
    o = oracle.Ctx.from_config(cfg)
    g = S.rng(seed)
    nk = len(cfg.q) + len(cfg.p)
    evk = np.stack([S.uniform_limbs(g, o.primes, o.n) for _ in range(2 * cfg.dnum)]).reshape(cfg.dnum, 2, nk, o.n)
    c0 = S.uniform_limbs(g, cfg.q[: level + 1], o.n)
    c1 = S.uniform_limbs(g, cfg.q[: level + 1], o.n)

    def one():
        t = time.perf_counter()
        o.keyswitch(c0, c1, evk, level)
        return time.perf_counter() - t
    return one


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def cpu_baseline(cfg, level, budget_s=20.0):
    """The oracle as it stands on the host: all cores (OpenMP over limbs / coefficients), then one KeySwitch
    single-threaded (SURVEY.md §8(d) oracle timing)."""
    import oracle
    one = oracle_ks_timer(cfg, level, 7)
    ts = [one()]
    while sum(ts) < budget_s * 0.5 and len(ts) < 10:
        ts.append(one())
    prev = oracle.set_num_threads(1)
    try:
        t1 = one()
    finally:
        oracle.set_num_threads(prev)
    return {"value": len(ts) / sum(ts), "unit": "KeySwitch/s", "cores": cpu_cores(), "kind": "oracle",
            "cpu_model": cpu_model(),
            "single_thread": {"value": 1.0 / t1, "unit": "KeySwitch/s", "cores": 1, "seconds": t1},
            "sample": f"{len(ts)} full KeySwitches of {cfg.name} at level {level} on {cpu_cores()} threads "
                      f"(oracle/oracle.c, %-on-u128, OpenMP over limbs), {sum(ts):.1f} s; then 1 KeySwitch on 1 "
                      f"thread, {t1:.1f} s"}


def run_reference(args, cfg, level):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    one = oracle_ks_timer(cfg, level, 7)
    budget = 150.0
    t_w = one()                                   # first warm-up step also sizes the run
    for _ in range(max(0, min(args.warmup, 3) - 1)):
        one()
    k = max(1, min(args.steps, int(budget / max(t_w, 1e-3))))
    ts = [one() for _ in range(k)]
    v = k / sum(ts)
    line = {"metric": METRIC, "value": v, "unit": "KeySwitch/s", "n_gpus": args.gpus, "steps": k,
            "warmup": min(args.warmup, 3), "ms_per_step": 1e3 * sum(ts) / k, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": workload_desc(cfg, level), "parallelism": "cpu oracle, rank 0 only"},
            "cpu_baseline": {"value": v, "unit": "KeySwitch/s", "kind": "oracle", "cores": cpu_cores(),
                             "sample": f"{k} full KeySwitches (steps capped at {budget:.0f} s of CPU time; "
                                       f"requested {args.steps})"},
            "e2e": {"value": v, "unit": "KeySwitch/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------------------- workloads
class KSWorkload:
    """C1 / C2 / C4 (unsharded): one relinearisation KeySwitch per step, rotating (ct, key) sets."""
    unit = "KeySwitch/s"
    scaling = "weak"

    def __init__(self, H, ctx, cfg, level, nsets, dev, seed, sid, conc=1, key="plain"):
        import torch
        self.H, self.ctx, self.cfg, self.level, self.sid = H, ctx, cfg, level, sid
        nsets = max(nsets, conc)
        self.sets = make_sets(cfg, level, nsets, dev, seed)
        self.key = key
        if key == "prepared":   # once per key at load time (include/hks.h hks_evk_prepare); dumps keep the raw key
            for s in self.sets:
                s["evk_raw"] = s["evk"]
                s["evk"] = H.evk_prepare(ctx, s["evk"], out=torch.empty_like(s["evk"]), stream=sid)
            torch.cuda.synchronize()
        self.conc = conc
        self.wss = [ctx.workspace(H.OP_KEYSWITCH, level) for _ in range(conc)]
        self.ws = self.wss[0]
        self.streams = [torch.cuda.Stream(dev) for _ in range(conc)] if conc > 1 else []
        self.units = conc
        self.nsets = nsets

    e2e_units = 1   # the e2e pipeline moves one ciphertext per step

    def step1(self, i):
        s = self.sets[i % len(self.sets)]
        self.H.keyswitch(self.ctx, s["c0"], s["c1"], self.level, s["evk"], s["out0"], s["out1"], self.ws, self.sid)

    def step(self, i):
        """One batch: `conc` KeySwitches of distinct (ct, key) sets, forked onto their own streams from the
        current stream and joined back (inside a CUDA graph: `conc` parallel branches)."""
        if self.conc == 1:
            s = self.sets[i % len(self.sets)]
            self.H.keyswitch(self.ctx, s["c0"], s["c1"], self.level, s["evk"], s["out0"], s["out1"], self.ws, self.sid)
            return
        import torch
        cur = torch.cuda.current_stream()
        for st in self.streams:
            st.wait_stream(cur)
        for j, st in enumerate(self.streams):
            s = self.sets[(i * self.conc + j) % len(self.sets)]
            self.H.keyswitch(self.ctx, s["c0"], s["c1"], self.level, s["evk"], s["out0"], s["out1"], self.wss[j],
                             st.cuda_stream)
        for st in self.streams:
            cur.wait_stream(st)

    def alg_bytes(self):
        c, l = self.cfg, self.level
        return self.conc * (4 * (l + 1) + 2 * c.beta(l) * (l + 1 + c.K)) * c.n * 8

    def l2_note(self):
        c, l = self.cfg, self.level
        b = self.nsets * (2 * c.dnum * (c.L + 1 + c.K) + 2 * (l + 1)) * c.n * 8
        rel = ">" if b > 4 * L2_BYTES else "<="
        return f"{self.nsets} rotating (ct, key) sets, {b / 2**20:.0f} MiB {rel} 4x the {l2_str()}"

    def dump(self, d, rank):
        s = self.sets[0]
        self.step1(0)
        import torch
        torch.cuda.synchronize()
        save_npy(d, rank, level=self.level, c0=s["c0"], c1=s["c1"], evk=s.get("evk_raw", s["evk"]), out0=s["out0"],
                 out1=s["out1"])

    # e2e: every step copies its ciphertext (c0, c1) H2D from pinned host memory, runs the KeySwitch
    # and copies (out0, out1) D2H.  Three streams pipeline step i's H2D, step i-1's KeySwitch and
    # step i-2's D2H (PCIe is full duplex), with events ordering each step's three stages.
    def e2e_setup(self):
        import torch
        dev = self.sets[0]["c0"].device
        self.NB = 3
        self.hin = [{k: self.sets[i % len(self.sets)][k].cpu().pin_memory() for k in ("c0", "c1")}
                    for i in range(2)]
        self.din = [{k: torch.empty_like(self.sets[0][k]) for k in ("c0", "c1")} for _ in range(self.NB)]
        self.dout = [{k: torch.empty_like(self.sets[0][k]) for k in ("out0", "out1")} for _ in range(self.NB)]
        self.hout = [{k: torch_empty_pinned_like(self.sets[0][k]) for k in ("out0", "out1")} for _ in range(self.NB)]
        self.s_in, self.s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        self.s_cmp = torch.cuda.current_stream(dev)
        self.ev_in = [torch.cuda.Event() for _ in range(self.NB)]
        self.ev_cmp = [torch.cuda.Event() for _ in range(self.NB)]
        self.ev_out = [torch.cuda.Event() for _ in range(self.NB)]
        io = 2 * (self.level + 1) * self.cfg.n * 8
        return io, io

    def e2e_step(self, i):
        import torch
        b = i % self.NB
        h, d, o, ho = self.hin[i % 2], self.din[b], self.dout[b], self.hout[b]
        s = self.sets[i % len(self.sets)]
        with torch.cuda.stream(self.s_in):
            self.s_in.wait_event(self.ev_cmp[b])          # buffer b's previous KeySwitch has read it
            d["c0"].copy_(h["c0"], non_blocking=True)
            d["c1"].copy_(h["c1"], non_blocking=True)
            self.ev_in[b].record(self.s_in)
        self.s_cmp.wait_event(self.ev_in[b])
        self.s_cmp.wait_event(self.ev_out[b])             # previous D2H of buffer b is done
        self.H.keyswitch(self.ctx, d["c0"], d["c1"], self.level, s["evk"], o["out0"], o["out1"], self.ws,
                         self.s_cmp.cuda_stream)
        self.ev_cmp[b].record(self.s_cmp)
        with torch.cuda.stream(self.s_out):
            self.s_out.wait_event(self.ev_cmp[b])
            ho["out0"].copy_(o["out0"], non_blocking=True)
            ho["out1"].copy_(o["out1"], non_blocking=True)
            self.ev_out[b].record(self.s_out)

    def e2e_streams(self):
        return self.s_in, self.s_out


class C4ShardWorkload:
    """C4 (BASELINE.json configs[3]): ONE KeySwitch per step with the RNS limbs sharded over the ranks
    (SURVEY.md §8(e) item 2).  mode "nccl": shard.ShardedKeySwitch, two all_gather_into_tensor per
    KeySwitch; mode "peer": shard.PeerShardedKeySwitch, base conversions read the peers' limbs over NVLink
    (symmetric memory), no all-gather.  At world 1 the exchange degenerates to the rank's own buffer."""
    unit = "KeySwitch/s"
    scaling = "strong"
    graphable = False      # collectives / symmetric-memory barriers: timed as direct calls

    def __init__(self, H, ctx, cfg, level, nsets, dev, seed, sid, world, rank, mode):
        import torch
        from paper_2507_04775_b200 import shard
        self.H, self.ctx, self.cfg, self.level, self.sid, self.mode = H, ctx, cfg, level, sid, mode
        self.world, self.rank = world, rank
        self.units = 1
        self.nsets = nsets
        if mode == "peer":
            if world > 1:
                self.ks = shard.PeerShardedKeySwitch(ctx, level, world, rank, dev)
            else:
                s0 = H.shard_query(ctx, level, 1, 0)
                ys = [torch.zeros((s0.q_pad, cfg.n), dtype=torch.int64, device=dev)]
                yps = [torch.zeros((2 * s0.p_pad, cfg.n), dtype=torch.int64, device=dev)]
                self.ks = shard.PeerShardedKeySwitch(ctx, level, 1, 0, dev, sim_ysend=ys, sim_ypsend=yps)
        elif mode == "a2a":
            def a2a_gloo(out, inp):      # HKS_BENCH_BACKEND=gloo (logic check): exchange through host tensors
                import torch.distributed as dist
                o = torch.empty(out.shape, dtype=out.dtype)
                dist.all_to_all_single(o, inp.cpu())
                out.copy_(o)
            fn = (lambda o, i: o.copy_(i)) if world == 1 else (
                a2a_gloo if os.environ.get("HKS_BENCH_BACKEND", "nccl") != "nccl" else None)
            self.ks = shard.A2AShardedKeySwitch(ctx, level, world, rank, dev, a2a_fn=fn)
        elif mode == "pipe":
            self.ks = shard.PipelinedShardedKeySwitch(ctx, level, world, rank, dev,
                                                      deliver_fn=None if world > 1 else (lambda j, runs, yall: None),
                                                      gather_fn=None if world > 1 else (lambda o, i: o.copy_(i)))
        else:
            self.ks = shard.ShardedKeySwitch(ctx, level, world, rank, dev,
                                             gather_fn=None if world > 1 else (lambda o, i: o.copy_(i)))
        info = self.ks.info
        g = torch.Generator(device=dev)
        g.manual_seed(seed)
        n = cfg.n
        q_own = list(cfg.q[info.q_lo:info.q_lo + info.nq_act])
        key_pr = list(cfg.q[info.q_lo:info.q_hi]) + list(cfg.p[info.p_lo:info.p_hi])

        def limbs(pr):
            t = torch.empty((len(pr), n), dtype=torch.int64, device=dev)
            for i, q in enumerate(pr):
                t[i] = torch.randint(0, int(q), (n,), generator=g, device=dev, dtype=torch.int64)
            return t

        self.sets = []
        for _ in range(nsets):
            c0, c1 = limbs(q_own), limbs(q_own)
            evk = torch.stack([limbs(key_pr) for _ in range(2 * cfg.dnum)]).reshape(cfg.dnum, 2, len(key_pr), n)
            self.sets.append({"c0": c0, "c1": c1, "evk": evk, "out0": torch.empty_like(c0),
                              "out1": torch.empty_like(c1)})

    def step(self, i):
        import torch
        s = self.sets[i % len(self.sets)]
        self.ks(s["c0"], s["c1"], s["evk"], s["out0"], s["out1"], self.sid)

    def alg_bytes(self):
        """one sharded KeySwitch per step: this rank's share of its algorithmic bytes"""
        c, l = self.cfg, self.level
        return (4 * (l + 1) + 2 * c.beta(l) * (l + 1 + c.K)) * c.n * 8 / self.world

    def l2_note(self):
        c, l = self.cfg, self.level
        b = self.nsets * (2 * c.dnum * (c.L + 1 + c.K) + 2 * (l + 1)) * c.n * 8 / self.world
        return (f"{self.nsets} rotating (ct, key) sets, {b / 2**20:.0f} MiB per rank ({l2_str()}); limbs sharded over "
                f"{self.world} rank(s), exchange: " + {"nccl": "NCCL all-gathers", "pipe": "per-digit broadcasts "
                                                        "overlapped with BConv + all-gather",
                                                        "a2a": "four all-to-alls, coefficient-sharded BConv",
                                                        "peer": "peer loads in BConv"}[self.mode])

    def dump(self, d, rank):
        import torch
        s = self.sets[0]
        self.step(0)
        torch.cuda.synchronize()
        i = self.ks.info
        save_npy(d, rank, level=self.level, world=self.world, q_lo=i.q_lo, q_hi=i.q_hi, p_lo=i.p_lo, p_hi=i.p_hi,
                 nq_act=i.nq_act, c0=s["c0"], c1=s["c1"], evk=s["evk"], out0=s["out0"], out1=s["out1"])


class C3Workload:
    """C3: 8 ciphertexts x 8 hoisted rotations, ciphertexts sharded over ranks (keys replicated)."""
    unit = "rotation-KeySwitch/s"
    scaling = "strong"

    def __init__(self, H, ctx, cfg, level, world, rank, dev, seed, sid):
        import torch
        self.H, self.ctx, self.cfg, self.level, self.sid = H, ctx, cfg, level, sid
        nct_total, self.nrot = 8, 8
        assert nct_total % world == 0, "C3 shards 8 ciphertexts: world size must divide 8"
        self.nct = nct_total // world
        self.galois = [S.galois_rot(r, cfg.log_n) for r in range(1, self.nrot + 1)]
        keysets = make_sets(cfg, level, self.nrot, dev, seed)            # one key per rotation
        self.evks = [k["evk"] for k in keysets]
        cts = make_sets(cfg, level, self.nct, dev, seed + 7)
        for k in keysets:
            del k["c0"], k["c1"], k["out0"], k["out1"]
        self.cts = [(c["c0"], c["c1"]) for c in cts]
        shape = cts[0]["c0"].shape
        self.out0 = [[torch.empty(shape, dtype=torch.int64, device=dev) for _ in range(self.nrot)] for _ in range(self.nct)]
        self.out1 = [[torch.empty(shape, dtype=torch.int64, device=dev) for _ in range(self.nrot)] for _ in range(self.nct)]
        self.ws = H.rotate_hoisted_batch_workspace(ctx, self.nct, level)
        self.units = self.nct * self.nrot
        self.c0s = [c[0] for c in self.cts]
        self.c1s = [c[1] for c in self.cts]
        self.flat0 = [o for c in range(self.nct) for o in self.out0[c]]
        self.flat1 = [o for c in range(self.nct) for o in self.out1[c]]

    def step(self, i):
        # one hoisted ModUp per ciphertext; per rotation key one key product over all of the rank's
        # ciphertexts (each key word loaded once) and one batched ModDown
        self.H.rotate_hoisted_batch(self.ctx, self.c0s, self.c1s, self.level, self.galois, self.evks, self.flat0,
                                    self.flat1, self.ws, self.sid)

    def alg_bytes(self):
        c, l = self.cfg, self.level
        key = 2 * c.beta(l) * (l + 1 + c.K) * c.n * 8
        ct = 2 * (l + 1) * c.n * 8
        return self.nrot * key + self.nct * ct + self.units * ct     # keys once, ct in, rotated cts out

    def l2_note(self):
        c = self.cfg
        return f"8 rotation keys ({8 * 2 * c.dnum * (c.L + 1 + c.K) * c.n * 8 / 2**20:.0f} MiB) > 4x the {l2_str()}"

    def dump(self, d, rank):
        """ciphertext 0 of this rank with rotations 0 and nrot - 1 (their keys and outputs)"""
        import torch
        self.step(0)
        torch.cuda.synchronize()
        r = [0, self.nrot - 1]
        save_npy(d, rank, level=self.level, galois=[self.galois[k] for k in r], c0=self.c0s[0], c1=self.c1s[0],
                 evk=torch.stack([self.evks[k] for k in r]), out0=torch.stack([self.out0[0][k] for k in r]),
                 out1=torch.stack([self.out1[0][k] for k in r]))


class C5Workload:
    """C5 = BOOT_SHAPE v2 on one ciphertext per rank (replicas): the bootstrapping schedule of
    SURVEY.md 8(d) built from the real operations (reading 14):
      CoeffToSlot: 3 BSGS linear transforms (n1 = n2 = 8: 7 hoisted baby + 7 giant rotations, 64
                   plaintext diagonals) at l = 29, 28, 27, each followed by Rescale;
      conjugation KS at l = 26;
      EvalMod stand-in: 12 x (HMult + Rescale) at l = 26 .. 15;
      SlotToCoeff: 3 BSGS transforms + Rescale at l = 14, 13, 12.
    97 KeySwitches per sequence (3*14 + 1 + 12 + 3*14)."""
    unit = "sequences/s"
    scaling = "weak"

    def __init__(self, H, ctx, cfg, dev, seed, sid):
        import torch
        self.H, self.ctx, self.cfg, self.sid = H, ctx, cfg, sid
        L, n = cfg.L, cfg.n
        self.n1 = self.n2 = 8
        self.baby = [S.galois_rot(r, cfg.log_n) for r in range(1, 8)]
        self.giant = [S.galois_rot(8 * r, cfg.log_n) for r in range(1, 8)]
        self.conj = S.GALOIS_CONJ(cfg.log_n)
        keys = make_sets(cfg, L, 16, dev, seed)
        self.kb = [keys[i]["evk"] for i in range(7)]
        self.kg = [keys[7 + i]["evk"] for i in range(7)]
        self.krelin, self.kconj = keys[14]["evk"], keys[15]["evk"]
        for k in keys:
            del k["c0"], k["c1"], k["out0"], k["out1"]
        g = torch.Generator(device=dev)
        g.manual_seed(seed + 5)
        q = torch.tensor([int(v) for v in cfg.q], dtype=torch.int64, device=dev).view(-1, 1)
        # 64 seeded diagonals [L+1][N] (uniform residues), sliced to each stage's level
        self.pts = [torch.randint(0, 2 ** 62, (L + 1, n), generator=g, device=dev, dtype=torch.int64) % q
                    for _ in range(self.n1 * self.n2)]
        ct = make_sets(cfg, L, 2, dev, seed + 3)
        self.c0, self.c1 = ct[0]["c0"], ct[0]["c1"]
        self.d0, self.d1 = ct[1]["c0"], ct[1]["c1"]                      # second HMult operand
        mk = lambda: torch.empty((L + 1, n), dtype=torch.int64, device=dev)
        self.a0, self.a1 = mk(), mk()
        self.ws_lt = H.linear_transform_workspace(ctx, L, self.n1)
        self.ws_ks = ctx.workspace(H.OP_HMULT, L)
        self.ws_rs = ctx.workspace(H.OP_RESCALE, L, 1)
        self.units = 1
        self.ks_per_seq = 97

    def _rescale(self, x0, x1, level, out0, out1):
        """Rescale (x0, x1) at level -> (out0, out1) at level - 1, one polynomial per call."""
        H, c, s = self.H, self.ctx, self.sid
        H.rescale(c, x0[: level + 1], 1, level, out0[:level], self.ws_rs, s)
        H.rescale(c, x1[: level + 1], 1, level, out1[:level], self.ws_rs, s)

    def _lt(self, level):
        H, c, s = self.H, self.ctx, self.sid
        l1 = level + 1
        H.linear_transform(c, self.c0[:l1], self.c1[:l1], level, self.n1, self.n2, self.baby, self.kb, self.giant,
                           self.kg, [p[:l1] for p in self.pts], self.a0[:l1], self.a1[:l1], self.ws_lt, s)
        self._rescale(self.a0, self.a1, level, self.c0, self.c1)

    def step(self, i):
        H, c, s, L = self.H, self.ctx, self.sid, self.cfg.L
        for level in (L, L - 1, L - 2):                                                    # CoeffToSlot
            self._lt(level)
        lv = L - 3
        H.rotate_hoisted(c, self.c0[: lv + 1], self.c1[: lv + 1], lv, [self.conj], [self.kconj],
                         [self.a0[: lv + 1]], [self.a1[: lv + 1]], self.ws_ks, s)        # conjugation
        for level in range(L - 3, L - 15, -1):                                             # EvalMod stand-in
            l1 = level + 1
            H.hmult(c, self.c0[:l1], self.c1[:l1], self.d0[:l1], self.d1[:l1], level, self.krelin,
                    self.a0[:l1], self.a1[:l1], self.ws_ks, s)
            self._rescale(self.a0, self.a1, level, self.c0, self.c1)
        for level in (L - 15, L - 16, L - 17):                                             # SlotToCoeff
            self._lt(level)

    def ops(self, timeit):
        """one BSGS linear transform (n1 = n2 = 8, 14 KeySwitches) at l = L, timed alone"""
        L, l1 = self.cfg.L, self.cfg.L + 1
        H, c, s = self.H, self.ctx, self.sid
        t = timeit(lambda i: H.linear_transform(c, self.c0, self.c1, L, 8, 8, self.baby, self.kb, self.giant, self.kg,
                                                self.pts, self.a0, self.a1, self.ws_lt, s), 10)
        return {"linear_transform_bsgs_8x8": {"us": 1e3 * t, "per_s": 1e3 / t, "keyswitch_per_s": 14e3 / t,
                                              "level": L}}

    def alg_bytes(self):
        c = self.cfg
        ks = lambda l: (4 * (l + 1) + 2 * c.beta(l) * (l + 1 + c.K)) * c.n * 8
        rs = lambda l: (4 * l + 2) * c.n * 8
        wsum = lambda l: 8 * (3 * 8 + 2) * (l + 1) * c.n * 8
        tot = 0
        for l in [c.L, c.L - 1, c.L - 2, c.L - 15, c.L - 16, c.L - 17]:
            tot += 14 * ks(l) + wsum(l) + rs(l)
        tot += ks(c.L - 3)
        for l in range(c.L - 3, c.L - 15, -1):
            tot += ks(l) + 4 * (l + 1) * c.n * 8 + rs(l)
        return tot

    def l2_note(self):
        c = self.cfg
        return (f"16 keys ({16 * 2 * c.dnum * (c.L + 1 + c.K) * c.n * 8 / 1e9:.2f} GB) + 64 diagonals "
                f"({64 * (c.L + 1) * c.n * 8 / 1e9:.2f} GB) >> the {l2_str()}")


def save_npy(d, rank, **kw):
    """one rank's dump: tensors as uint64 .npy, scalars / lists in meta.json (bench.py --dump)"""
    import numpy as np
    out = os.path.join(d, f"rank{rank}")
    os.makedirs(out, exist_ok=True)
    meta = {}
    for k, v in kw.items():
        if hasattr(v, "cpu"):
            np.save(os.path.join(out, k + ".npy"), v.cpu().numpy().view(np.uint64))
        else:
            meta[k] = v
    with open(os.path.join(out, "meta.json"), "w") as f:
        json.dump(meta, f)


def torch_empty_pinned_like(t):
    import torch
    return torch.empty(t.shape, dtype=t.dtype, device="cpu").pin_memory()


# ---------------------------------------------------------------------------------------------- main
def main():
    args = parse()
    cfg = S.config(args.config)
    level = cfg.L if args.level is None else args.level
    if args.impl == "reference":
        run_reference(args, cfg, level)
        return

    import torch
    import torch.distributed as dist
    from paper_2507_04775_b200 import hks as H

    global L2_BYTES
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # HKS_BENCH_BACKEND=gloo: several ranks sharing the visible GPUs (a check of the multi-rank logic --
    # sharding, barriers, max over ranks, one line from rank 0 -- on a one-GPU box; never a bench number)
    backend = os.environ.get("HKS_BENCH_BACKEND", "nccl")
    local = local % max(torch.cuda.device_count(), 1) if backend != "nccl" else local
    torch.cuda.set_device(local)
    dev = f"cuda:{local}"
    L2_BYTES = int(getattr(torch.cuda.get_device_properties(local), "L2_cache_size", L2_BYTES)) or L2_BYTES
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device(dev))
        else:
            dist.init_process_group(backend)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world > 1:
            t = torch.tensor([x], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return float(t.item())
        return x

    ctx = H.Context.from_config(cfg, local)
    stream = torch.cuda.current_stream()
    sid = stream.cuda_stream
    seed = cfg.seed * 1000 + rank
    shard_mode = args.shard if args.shard != "auto" else ("nccl" if cfg.name == "C4" and world > 1 else "none")
    if shard_mode != "none" and cfg.name != "C4":
        raise SystemExit("--shard nccl|peer applies to --config C4 (limb sharding)")
    if shard_mode != "none":
        wl = C4ShardWorkload(H, ctx, cfg, level, args.sets, dev, seed, sid, world, rank, shard_mode)
    elif cfg.name == "C3":
        wl = C3Workload(H, ctx, cfg, level, world, rank, dev, seed, sid)
    elif cfg.name == "C5":
        wl = C5Workload(H, ctx, cfg, dev, seed, sid)
    else:
        conc = args.streams or {"C1": 8, "C2": 3, "C4": 2}.get(cfg.name, 1)
        wl = KSWorkload(H, ctx, cfg, level, args.sets, dev, seed, sid, conc, args.key)

    for i in range(args.warmup):
        wl.step(i)
    torch.cuda.synchronize()

    # CUDA graphs: each distinct step (one per rotating input set) is captured once from the same
    # C-ABI calls and replayed; the library's launch counter during capture gives the kernels per
    # replay (gpu_launches counts the kernels the timed region executes either way)
    period = len(wl.sets) if hasattr(wl, "sets") else 1
    graphs, glaunch = [], []
    if not args.no_graph and getattr(wl, "graphable", True):
        for i in range(period):
            g = torch.cuda.CUDAGraph()
            sid0 = wl.sid
            n_c = H.launch_count()
            with torch.cuda.graph(g, capture_error_mode="thread_local"):
                wl.sid = torch.cuda.current_stream().cuda_stream
                wl.step(i)
            wl.sid = sid0
            glaunch.append(H.launch_count() - n_c)
            graphs.append(g)
        for i in range(args.warmup):
            graphs[i % period].replay()
        torch.cuda.synchronize()

    def tstep(i):
        if graphs:
            graphs[i % period].replay()
        else:
            wl.step(i)

    barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n0 = H.launch_count()
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for i in range(args.steps):
            tstep(i)
        ev1.record(stream)
        ev1.synchronize()
    launches = H.launch_count() - n0 + sum(glaunch[i % period] for i in range(args.steps)) if graphs else \
        H.launch_count() - n0
    torch.cuda.synchronize()
    barrier()
    ms = max_over_ranks(ev0.elapsed_time(ev1))
    total_units = world * wl.units if wl.scaling == "weak" else 8 * wl.nrot if cfg.name == "C3" else wl.units
    value = total_units * args.steps / (ms / 1e3)

    hbm_peak, peak_src = peaks()
    extra = {}
    if not args.quick:
        # ---- per-step distribution (SURVEY 8(d) timing protocol: median, p10, p90), own pass so
        # the per-step events do not perturb the timed region above
        nd = max(1, min(args.steps, 200))
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(nd + 1)]
        evs[0].record(stream)
        for i in range(nd):
            tstep(i)
            evs[i + 1].record(stream)
        evs[-1].synchronize()
        per = sorted(evs[i].elapsed_time(evs[i + 1]) for i in range(nd))
        q = lambda f: per[min(nd - 1, int(f * nd))]
        extra["step_ms"] = {"p10": q(0.1), "median": q(0.5), "p90": q(0.9), "steps": nd}

        # ---- configs[1] as stated: ONE ciphertext per step (no concurrent batch), same sets, graphs, timing
        if isinstance(wl, KSWorkload) and wl.conc > 1:
            g1 = []
            if graphs:
                for i in range(len(wl.sets)):
                    g = torch.cuda.CUDAGraph()
                    ws0 = wl.ws
                    with torch.cuda.graph(g, capture_error_mode="thread_local"):
                        s_ = wl.sets[i]
                        H.keyswitch(ctx, s_["c0"], s_["c1"], level, s_["evk"], s_["out0"], s_["out1"], ws0,
                                    torch.cuda.current_stream().cuda_stream)
                    g1.append(g)
            run1 = (lambda i: g1[i % len(g1)].replay()) if g1 else wl.step1
            for i in range(max(3, args.warmup)):
                run1(i)
            torch.cuda.synchronize()
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for i in range(args.steps):
                run1(i)
            e1.record(stream)
            e1.synchronize()
            t1 = max_over_ranks(e0.elapsed_time(e1)) / args.steps
            extra["single_ciphertext"] = {"value": world / (t1 * 1e-3), "unit": wl.unit, "ms_per_keyswitch": t1,
                                          "note": "one KeySwitch per step on one stream (BASELINE configs[1] as "
                                                  "stated); `value` batches --streams ciphertexts per step"}

        # ---- per-kernel breakdown: CUDA events recorded by libhks around each launch, same stream
        H.prof_enable(True)
        nprof = max(1, min(args.steps, 100 if cfg.name not in ("C3", "C5") else 5))
        for i in range(nprof):   # kernels of one KeySwitch at a time (no concurrent-stream overlap in the events)
            getattr(wl, "step1", wl.step)(i)
        prof = H.prof_read()
        H.prof_enable(False)
        tot = sum(v[1] for v in prof.values())
        mpeak, mpeak_src = mul_peak()
        kern = {k: {"launches_per_step": v[0] / nprof, "ms_per_step": v[1] / nprof, "share": v[1] / tot,
                    "avg_launch_us": 1e3 * v[1] / v[0], "alg_bytes_per_launch": v[2] / v[0],
                    "achieved_gbs": (v[2] / v[0]) / (1e-3 * v[1] / v[0]) / 1e9,
                    "alg_muls_per_launch": v[3] / v[0],
                    "achieved_tmul": (v[3] / v[0]) / (1e-3 * v[1] / v[0]) / 1e12}
                for k, v in prof.items()}
        for k in kern.values():
            k["hbm_frac"] = k["achieved_gbs"] / hbm_peak
            k["alu_frac"] = k["achieved_tmul"] * 1e12 / mpeak
        dom = max(kern, key=lambda k: kern[k]["share"])
        d = kern[dom]
        traffic = None
        tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tpath):
            with open(tpath) as f:
                traffic = json.load(f).get(cfg.name, {}).get(dom)
        hbm = {"kernel": dom, "bound": "hbm", "achieved": d["achieved_gbs"], "peak": hbm_peak, "unit": "GB/s",
               "frac": d["hbm_frac"], "traffic": traffic, "peak_source": peak_src, "share_of_step": d["share"]}
        alu = {"kernel": dom, "bound": "alu", "achieved": d["achieved_tmul"], "peak": mpeak / 1e12,
               "unit": "T int-mul32x32/s", "frac": d["alu_frac"], "traffic": traffic, "peak_source": mpeak_src,
               "share_of_step": d["share"],
               "work": "algorithmic 32x32->64 partial products: 4 per exact 60x60-bit product, 7 per Shoup butterfly"}
        # the binding roofline of the dominant kernel is the one it is closer to
        extra["roofline"], extra["roofline_other"] = (alu, hbm) if d["alu_frac"] >= d["hbm_frac"] else (hbm, alu)
        extra["kernels"] = kern
        alg = wl.alg_bytes()
        extra["step_hbm"] = {"alg_bytes": alg, "achieved_gbs": alg / (ms / args.steps * 1e-3) / 1e9,
                             "frac": alg / (ms / args.steps * 1e-3) / 1e9 / hbm_peak}
        # ---- step-level roofline: max(T_HBM, T_INT, T_tensor) / T_measured for the unit the
        # profile pass ran (one KeySwitch for C1/C2/C4, one step otherwise); the pipes overlap, so the bound is
        # the largest of the three
        per_ks = isinstance(wl, KSWorkload)
        t_unit = (ms / args.steps) * 1e-3 / (wl.conc if per_ks else 1)
        b_unit = alg / (wl.conc if per_ks else 1)
        m_unit = sum(v[3] for v in prof.values()) / nprof
        tc_ops = 0.0
        if per_ks and prof.get("bconv", (0, 0, 0, 1))[3] == 0:      # conversions ran on the tensor cores
            c_, l_ = cfg, level
            macs = sum((min((j + 1) * c_.alpha, l_ + 1) - j * c_.alpha) * (l_ + 1 + c_.K - (min((j + 1) * c_.alpha, l_ + 1) - j * c_.alpha))
                       for j in range(c_.beta(l_))) + 2 * c_.K * (l_ + 1)
            tc_ops = 2.0 * 64 * macs * c_.n          # u8 products: 8 bytes x 8 byte columns per 60-bit MAC
        tpk, tpk_src = tensor_peak()
        tb = {"hbm": b_unit / (hbm_peak * 1e9), "int": m_unit / mpeak, "tensor": tc_ops / tpk}
        bound = max(tb, key=tb.get)
        extra["step_roofline"] = {"unit": "KeySwitch" if per_ks else "step", "t_measured_us": 1e6 * t_unit,
                                  "t_hbm_us": 1e6 * tb["hbm"], "t_int_us": 1e6 * tb["int"],
                                  "t_tensor_us": 1e6 * tb["tensor"], "bound": bound, "frac": tb[bound] / t_unit,
                                  "peaks": {"hbm": peak_src, "int": mpeak_src, "tensor": tpk_src}}

        # ---- NTT limbs/s: the ModUp NTT batch (beta(l+1+K) - (l+1) limbs), 4 buffers > L2
        beta = cfg.beta(level)
        nl = beta * (level + 1 + cfg.K) - (level + 1)
        prim = list(range(len(cfg.q) + len(cfg.p)))
        idx = [prim[i % len(prim)] for i in range(nl)]
        bufs = [torch.randint(0, int(cfg.p[-1]), (nl, cfg.n), device=dev, dtype=torch.int64) for _ in range(4)]
        for kind, fn in (("fwd", H.ntt_fwd), ("inv", H.ntt_inv)):
            for i in range(3):
                fn(ctx, bufs[i % 4], idx, sid)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            it = 40
            e0.record(stream)
            for i in range(it):
                fn(ctx, bufs[i % 4], idx, sid)
            e1.record(stream)
            e1.synchronize()
            t = e0.elapsed_time(e1) / it
            extra[f"ntt_{kind}_limbs_per_s"] = nl / (t * 1e-3) * world
            extra[f"ntt_{kind}_hbm_frac"] = 2 * nl * cfg.n * 8 / (t * 1e-3) / 1e9 / hbm_peak
        del bufs

        # ---- NEXT-1 ops at this level (Table 3 "HMult" / "Rescale" rows): fused HMult
        # (tensor + relinearisation) and Rescale of a 2-polynomial ciphertext, rotating the KS sets
        if isinstance(wl, KSWorkload) and level >= 1:
            ops = {}
            sets = wl.sets
            outs = [torch.empty_like(sets[0]["c0"]) for _ in range(2)]
            wsh = ctx.workspace(H.OP_HMULT, level)
            xs = [torch.stack([s["c0"], s["c1"]]) for s in sets]
            rout = torch.empty((2, level, cfg.n), dtype=torch.int64, device=dev)
            wsr = ctx.workspace(H.OP_RESCALE, level, 2)

            def hm(i):
                a, b = sets[i % len(sets)], sets[(i + 1) % len(sets)]
                H.hmult(ctx, a["c0"], a["c1"], b["c0"], b["c1"], level, a["evk"], outs[0], outs[1], wsh, sid)

            def rs(i):
                H.rescale(ctx, xs[i % len(xs)], 2, level, rout, wsr, sid)

            # throughput mode: 8 ciphertexts relinearised with ONE key per call (key words read once
            # for the batch; hks_rotate_hoisted_batch with Galois element 1 = KeySwitch)
            NBT = 8
            bc0 = [sets[i % len(sets)]["c0"] for i in range(NBT)]
            bc1 = [sets[i % len(sets)]["c1"] for i in range(NBT)]
            bo0 = [torch.empty_like(bc0[0]) for _ in range(NBT)]
            bo1 = [torch.empty_like(bc0[0]) for _ in range(NBT)]
            wsb = H.rotate_hoisted_batch_workspace(ctx, NBT, level)

            def kb(i):
                H.rotate_hoisted_batch(ctx, bc0, bc1, level, [1], [sets[i % len(sets)]["evk"]], bo0, bo1, wsb, sid)

            for name, fn, it, nbytes in (
                    ("hmult", hm, 50, (6 * (level + 1) + 2 * cfg.beta(level) * (level + 1 + cfg.K)) * cfg.n * 8),
                    ("rescale", rs, 200, (2 * (level + 1) + 2 * level) * cfg.n * 8),
                    ("keyswitch_batch8_shared_key", kb, 20,
                     (NBT * 4 * (level + 1) + 2 * cfg.beta(level) * (level + 1 + cfg.K)) * cfg.n * 8)):
                for i in range(3):
                    fn(i)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                for i in range(it):
                    fn(i)
                e1.record(stream)
                e1.synchronize()
                t = e0.elapsed_time(e1) / it
                ops[name] = {"us": 1e3 * t, "per_s": 1e3 / t, "alg_bytes": nbytes,
                             "hbm_frac": nbytes / (t * 1e-3) / 1e9 / hbm_peak}
            ops["keyswitch_batch8_shared_key"]["keyswitch_per_s"] = NBT * ops["keyswitch_batch8_shared_key"]["per_s"]
            extra["ops"] = ops
            del xs, wsh, wsr, wsb, bo0, bo1

        if hasattr(wl, "ops"):
            def timeit(fn, it):
                for i in range(2):
                    fn(i)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                for i in range(it):
                    fn(i)
                e1.record(stream)
                e1.synchronize()
                return e0.elapsed_time(e1) / it
            extra["ops"] = wl.ops(timeit)

        # ---- e2e: through the public API from pinned host buffers, H2D + op + D2H per step
        if hasattr(wl, "e2e_setup"):
            h2d, d2h = wl.e2e_setup()
            e_steps = min(args.steps, 50)
            for i in range(3):
                wl.e2e_step(i)
            torch.cuda.synchronize()
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s_in, s_out = wl.e2e_streams()
            e0.record(s_in)
            for i in range(e_steps):
                wl.e2e_step(i)
            s_out.wait_stream(stream)
            e1.record(s_out)
            e1.synchronize()
            et = max_over_ranks(e0.elapsed_time(e1))
            extra["e2e"] = {"value": world * getattr(wl, "e2e_units", wl.units) * e_steps / (et / 1e3), "unit": wl.unit,
                            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": e_steps}

    if args.dump and hasattr(wl, "dump"):
        wl.dump(args.dump, rank)
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": wl.unit, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
                "scaling": wl.scaling, "vs_baseline": None, "dtype": "u64", "data": "synthetic",
                "config": {"workload": workload_desc(cfg, level), "N": cfg.n, "L": cfg.L, "K": cfg.K,
                           "dnum": cfg.dnum, "level": level,
                           "parallelism": (f"RNS limbs sharded over {world} GPU(s) ({shard_mode})"
                                           if shard_mode != "none" else
                                           f"{'replicas' if cfg.name == 'C5' else 'ciphertexts sharded'} over {world} GPU(s)"),
                           "l2": wl.l2_note(),
                           **({"batch": (f"{wl.conc} ciphertexts per step, each KeySwitched on its own CUDA stream"
                                         if wl.conc > 1 else "1 ciphertext per step")}
                              if isinstance(wl, KSWorkload) else {}),
                           **({"key": ("prepared once at load time (hks_evk_prepare: P^-1 on the Q limbs, folded "
                                       "into the ModDown conversion)" if wl.key == "prepared" else "as generated")}
                              if isinstance(wl, KSWorkload) else {})},
                "gpu_launches": launches, "clocks": clk.summary(),
                "launch_mode": (f"CUDA graph replay of the C-ABI calls ({glaunch[0]} kernels per step)" if graphs
                                else "direct C-ABI calls")}
        if cfg.name == "C5":
            line["keyswitch_per_s"] = value * wl.ks_per_seq
        line.update(extra)
        if "ntt_fwd_limbs_per_s" in extra:
            line["ntt_limbs_per_s"] = extra["ntt_fwd_limbs_per_s"]
        if world == 1 and not args.no_cpu_baseline and not args.quick and isinstance(wl, KSWorkload):
            line["cpu_baseline"] = cpu_baseline(cfg, level)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
