"""Limb-sharded KeySwitch across ranks (BASELINE.json configs[3]).

Each rank (one GPU) owns a contiguous slice of the chain limbs and of the special limbs
(`hks_shard_query`).  A KeySwitch is three library phases around two all-gathers that this module
issues with torch.distributed (NCCL over NVLink on the GPU box, gloo in CPU tests):

    A  ysend  = INTT(c1_loc) scaled                       -> all_gather -> yall
    B  acc    = KIP(NTT(BConv(yall)))  ; ypsend = INTT(acc_P)  -> all_gather -> ypall
    C  out    = (acc - NTT(BConv(ypall))) P^-1 (+ c0)

The collectives are ordinary NCCL all-gathers (`all_gather_into_tensor`, padded to equal chunks);
the math runs in libhks.  `gather_fn` can be replaced (tests use a local concatenation to simulate
several ranks on one device).
"""
from __future__ import annotations

from . import hks as H


class ShardPlan:
    """Host-side view of the ownership plan of every rank (computed by libhks)."""

    def __init__(self, ctx, level: int, world: int):
        self.level, self.world = level, world
        self.info = [H.shard_query(ctx, level, world, r) for r in range(world)]
        self.q_pad = self.info[0].q_pad
        self.p_pad = self.info[0].p_pad

    def q_slot(self, i: int) -> int:
        """Slot of chain limb i in the gathered y buffer [world][q_pad]."""
        for r, s in enumerate(self.info):
            if s.q_lo <= i < s.q_hi:
                return r * self.q_pad + (i - s.q_lo)
        raise IndexError(i)

    def p_slot(self, k: int, poly: int) -> int:
        """Slot of special limb k of polynomial `poly` in the gathered buffer [world][2][p_pad]."""
        for r, s in enumerate(self.info):
            if s.p_lo <= k < s.p_hi:
                return r * 2 * self.p_pad + poly * self.p_pad + (k - s.p_lo)
        raise IndexError(k)


class ShardedKeySwitch:
    """One rank's part of a limb-sharded KeySwitch at `level` (buffers allocated once)."""

    def __init__(self, ctx, level: int, world: int, rank: int, device, gather_fn=None):
        import torch
        self.ctx, self.level, self.world, self.rank = ctx, level, world, rank
        self.info = H.shard_query(ctx, level, world, rank)
        n = ctx.n
        s = self.info
        self.ysend = torch.zeros((s.q_pad, n), dtype=torch.int64, device=device)
        self.yall = torch.empty((world * s.q_pad, n), dtype=torch.int64, device=device)
        self.ypsend = torch.zeros((2 * s.p_pad, n), dtype=torch.int64, device=device)
        self.ypall = torch.empty((world * 2 * s.p_pad, n), dtype=torch.int64, device=device)
        self.acc = torch.empty((2 * (s.nq_act + s.p_hi - s.p_lo), n), dtype=torch.int64, device=device)
        self.ws = torch.empty((max(H.shard_workspace_bytes(ctx, level, world, rank) // 8, 1),), dtype=torch.int64,
                              device=device)
        self.gather = gather_fn or self._nccl_gather

    @staticmethod
    def _nccl_gather(out, inp):
        import torch.distributed as dist
        dist.all_gather_into_tensor(out, inp)

    def phase_a(self, c1_loc, stream=None):
        H.shard_ks_modup_in(self.ctx, self.level, self.world, self.rank, c1_loc, self.ysend, stream)

    def phase_b(self, c1_loc, evk_loc, stream=None):
        H.shard_ks_inner(self.ctx, self.level, self.world, self.rank, self.yall, c1_loc, evk_loc, self.acc,
                         self.ypsend, self.ws, stream)

    def phase_c(self, c0_loc, out0_loc, out1_loc, stream=None):
        H.shard_ks_moddown_out(self.ctx, self.level, self.world, self.rank, self.ypall, self.acc, c0_loc, out0_loc,
                               out1_loc, self.ws, stream)

    def __call__(self, c0_loc, c1_loc, evk_loc, out0_loc, out1_loc, stream=None):
        self.phase_a(c1_loc, stream)
        self.gather(self.yall, self.ysend)
        self.phase_b(c1_loc, evk_loc, stream)
        self.gather(self.ypall, self.ypsend)
        self.phase_c(c0_loc, out0_loc, out1_loc, stream)


def digit_segments(ctx, level: int, world: int):
    """Per digit j of `level`, the (owner rank, first slot, end slot) runs of its chain limbs in the gathered
    y buffer [world][q_pad][N] (slot of limb i = r * q_pad + i - q_lo(r)): one broadcast per run delivers the
    digit.  Host logic only (tests/test_shard.py checks it with gloo)."""
    infos = [H.shard_query(ctx, level, world, r) for r in range(world)]
    q_pad = infos[0].q_pad
    q = ctx.query(level)
    segs = []
    for j in range(q.beta):
        lo, hi = q.digit_lo[j], q.digit_hi[j]
        runs = []
        for r, s in enumerate(infos):
            a, b = max(lo, s.q_lo), min(hi, s.q_hi)
            if a < b:
                runs.append((r, r * q_pad + a - s.q_lo, r * q_pad + b - s.q_lo))
        segs.append(runs)
    return segs


class PipelinedShardedKeySwitch:
    """Limb-sharded KeySwitch with the first exchange delivered digit by digit and overlapped with the base
    conversions ("per-digit pipelined all-gather"): phase A writes this rank's scaled
    COEFF limbs straight into its own slots of the gathered buffer; every (digit, owner) run of chain limbs is
    then broadcast by its owner (NCCL over NVLink; async, on the process group's stream) and an event per digit
    records its arrival on an auxiliary stream; phase B (hks_shard_ks_inner_pipelined) waits on digit j's event
    only before digit j's conversion, so the conversion of one digit overlaps the transfer of the next.  No
    padding: a rank receives exactly the chain limbs it does not own.  The second exchange (P-parts of the
    accumulators) stays one all_gather_into_tensor.

    `deliver_fn(j, runs, yall)` replaces the broadcasts (simulated ranks on one GPU in the tests): it must enqueue
    the delivery of digit j on the current stream."""

    def __init__(self, ctx, level: int, world: int, rank: int, device, deliver_fn=None, gather_fn=None):
        import torch
        self.ctx, self.level, self.world, self.rank = ctx, level, world, rank
        self.info = H.shard_query(ctx, level, world, rank)
        s, n = self.info, ctx.n
        self.segments = digit_segments(ctx, level, world)
        self.yall = torch.zeros((world * s.q_pad, n), dtype=torch.int64, device=device)
        self.ysend = self.yall[rank * s.q_pad:(rank + 1) * s.q_pad]            # phase A output = own slots
        self.ypsend = torch.zeros((2 * s.p_pad, n), dtype=torch.int64, device=device)
        self.ypall = torch.empty((world * 2 * s.p_pad, n), dtype=torch.int64, device=device)
        self.acc = torch.empty((2 * (s.nq_act + s.p_hi - s.p_lo), n), dtype=torch.int64, device=device)
        self.ws = torch.empty((max(H.shard_workspace_bytes(ctx, level, world, rank) // 8, 1),), dtype=torch.int64,
                              device=device)
        self.aux = torch.cuda.Stream(device)
        self.events = [torch.cuda.Event() for _ in self.segments]
        self.deliver = deliver_fn
        self.gather = gather_fn or ShardedKeySwitch._nccl_gather

    def phase_a(self, c1_loc, stream=None):
        H.shard_ks_modup_in(self.ctx, self.level, self.world, self.rank, c1_loc, self.ysend, stream)

    def deliver_digits(self):
        """enqueue every digit's delivery; events[j] fires when digit j has arrived"""
        import torch
        if self.deliver is not None:
            cur = torch.cuda.current_stream()
            self.aux.wait_stream(cur)
            with torch.cuda.stream(self.aux):
                for j, runs in enumerate(self.segments):
                    self.deliver(j, runs, self.yall)
                    self.events[j].record(self.aux)
            return
        import torch.distributed as dist
        works = [[dist.broadcast(self.yall[lo:hi], src=r, async_op=True) for r, lo, hi in runs]
                 for runs in self.segments]
        with torch.cuda.stream(self.aux):
            for j, ws in enumerate(works):
                for w in ws:
                    w.wait()
                self.events[j].record(self.aux)

    def phase_b(self, c1_loc, evk_loc, stream=None):
        H.shard_ks_inner_pipelined(self.ctx, self.level, self.world, self.rank, self.yall, self.events, c1_loc, evk_loc,
                                   self.acc, self.ypsend, self.ws, stream)

    def phase_c(self, c0_loc, out0_loc, out1_loc, stream=None):
        H.shard_ks_moddown_out(self.ctx, self.level, self.world, self.rank, self.ypall, self.acc, c0_loc, out0_loc,
                               out1_loc, self.ws, stream)

    def __call__(self, c0_loc, c1_loc, evk_loc, out0_loc, out1_loc, stream=None):
        self.phase_a(c1_loc, stream)
        self.deliver_digits()
        self.phase_b(c1_loc, evk_loc, stream)
        self.gather(self.ypall, self.ypsend)
        self.phase_c(c0_loc, out0_loc, out1_loc, stream)


class A2AShardedKeySwitch:
    """Limb-sharded KeySwitch with coefficient-sharded base conversions: four
    all_to_all_single exchanges instead of two all-gathers.  Rank k converts coefficient chunk k (rows
    [k R / G, (k + 1) R / G)) of every limb, so it receives the chunk of every source limb and then its own
    converted limbs' chunks -- about 30 instead of 47 MiB per GPU at C4 / G = 8.  The math
    is in libhks (hks_shard_a2a_*); `a2a_fn(out, inp)` replaces the collective (simulated ranks in tests)."""

    def __init__(self, ctx, level: int, world: int, rank: int, device, a2a_fn=None):
        import torch
        self.ctx, self.level, self.world, self.rank = ctx, level, world, rank
        self.info = H.shard_query(ctx, level, world, rank)
        x = self.a2a_info = H.shard_a2a_query(ctx, level, world, rank)
        s, nc, G, n = self.info, x.chunk_words, world, ctx.n
        mk = lambda rows, cols: torch.zeros((rows, cols), dtype=torch.int64, device=device)
        self.ysend, self.yrecv = mk(G * s.q_pad, nc), mk(G * s.q_pad, nc)
        self.extsend, self.extrecv = mk(G * x.beta * x.n_pad, nc), mk(G * x.beta * x.n_pad, nc)
        self.ypsend, self.yprecv = mk(G * 2 * s.p_pad, nc), mk(G * 2 * s.p_pad, nc)
        self.convsend, self.convrecv = mk(G * 2 * x.nq_pad, nc), mk(G * 2 * x.nq_pad, nc)
        self.acc = torch.empty((2 * (s.nq_act + s.p_hi - s.p_lo), n), dtype=torch.int64, device=device)
        self.ws = torch.empty((max(H.shard_a2a_workspace_bytes(ctx, level, world, rank) // 8, 1),), dtype=torch.int64,
                              device=device)
        self.a2a = a2a_fn or self._nccl_a2a

    @staticmethod
    def _nccl_a2a(out, inp):
        import torch.distributed as dist
        dist.all_to_all_single(out, inp)

    def phase1(self, c1_loc, stream=None):
        H.shard_a2a_modup_in(self.ctx, self.level, self.world, self.rank, c1_loc, self.ysend, self.ws, stream)

    def phase2(self, stream=None):
        H.shard_a2a_bconv(self.ctx, self.level, self.world, self.rank, self.yrecv, self.extsend, stream)

    def phase3(self, c1_loc, evk_loc, stream=None):
        H.shard_a2a_inner(self.ctx, self.level, self.world, self.rank, self.extrecv, c1_loc, evk_loc, self.acc,
                          self.ypsend, self.ws, stream)

    def phase4(self, stream=None):
        H.shard_a2a_moddown_bconv(self.ctx, self.level, self.world, self.rank, self.yprecv, self.convsend, stream)

    def phase5(self, c0_loc, out0_loc, out1_loc, stream=None):
        H.shard_a2a_moddown_out(self.ctx, self.level, self.world, self.rank, self.convrecv, self.acc, c0_loc, out0_loc,
                                out1_loc, self.ws, stream)

    def __call__(self, c0_loc, c1_loc, evk_loc, out0_loc, out1_loc, stream=None):
        self.phase1(c1_loc, stream)
        self.a2a(self.yrecv, self.ysend)
        self.phase2(stream)
        self.a2a(self.extrecv, self.extsend)
        self.phase3(c1_loc, evk_loc, stream)
        self.a2a(self.yprecv, self.ypsend)
        self.phase4(stream)
        self.a2a(self.convrecv, self.convsend)
        self.phase5(c0_loc, out0_loc, out1_loc, stream)


class PeerShardedKeySwitch:
    """Limb-sharded KeySwitch with both exchanges fused into the base conversions:
    ysend / ypsend live in symmetric memory (torch.distributed._symmetric_memory, NVLink peer mappings),
    and phases B and C hand libhks the table of every rank's buffer address, so the BConv kernel loads
    each source limb straight from its owner -- no all-gather, no gathered copy, and each rank reads only
    the limbs its targets need.  Device-side barriers on the stream order the phases across ranks.

    Simulated ranks (tests, one GPU): pass `sim_ysend` / `sim_ypsend`, the lists of every rank's buffers;
    the caller then runs phase A of all ranks before phase B of any, and so on."""

    def __init__(self, ctx, level: int, world: int, rank: int, device, group=None, sim_ysend=None, sim_ypsend=None):
        import torch
        self.ctx, self.level, self.world, self.rank = ctx, level, world, rank
        self.info = H.shard_query(ctx, level, world, rank)
        s, n = self.info, ctx.n
        self.sim = sim_ysend is not None
        if self.sim:
            self.ysend, self.ypsend = sim_ysend[rank], sim_ypsend[rank]
            self.yptrs = [t.data_ptr() for t in sim_ysend]
            self.ypptrs = [t.data_ptr() for t in sim_ypsend]
        else:
            import torch.distributed as dist
            import torch.distributed._symmetric_memory as symm
            grp = group or dist.group.WORLD
            self.ysend = symm.empty((s.q_pad, n), dtype=torch.int64, device=device)
            self.ypsend = symm.empty((2 * s.p_pad, n), dtype=torch.int64, device=device)
            self._hy = symm.rendezvous(self.ysend, grp)
            self._hyp = symm.rendezvous(self.ypsend, grp)
            self.yptrs = list(self._hy.buffer_ptrs)
            self.ypptrs = list(self._hyp.buffer_ptrs)
        self.acc = torch.empty((2 * (s.nq_act + s.p_hi - s.p_lo), n), dtype=torch.int64, device=device)
        self.ws = torch.empty((max(H.shard_workspace_bytes(ctx, level, world, rank) // 8, 1),), dtype=torch.int64,
                              device=device)

    def barrier(self):
        """Stream-ordered barrier across ranks (no-op for simulated ranks)."""
        if not self.sim:
            self._hy.barrier(channel=0)

    def phase_a(self, c1_loc, stream=None):
        H.shard_ks_modup_in(self.ctx, self.level, self.world, self.rank, c1_loc, self.ysend, stream)

    def phase_b(self, c1_loc, evk_loc, stream=None):
        H.shard_ks_inner_peer(self.ctx, self.level, self.world, self.rank, self.yptrs, c1_loc, evk_loc, self.acc,
                              self.ypsend, self.ws, stream)

    def phase_c(self, c0_loc, out0_loc, out1_loc, stream=None):
        H.shard_ks_moddown_out_peer(self.ctx, self.level, self.world, self.rank, self.ypptrs, self.acc, c0_loc,
                                    out0_loc, out1_loc, self.ws, stream)

    def __call__(self, c0_loc, c1_loc, evk_loc, out0_loc, out1_loc, stream=None):
        self.phase_a(c1_loc, stream)
        self.barrier()          # every ysend written before any rank reads it
        self.phase_b(c1_loc, evk_loc, stream)
        self.barrier()          # every ypsend written (and every ysend read) before phase C / the next call
        self.phase_c(c0_loc, out0_loc, out1_loc, stream)
        self.barrier()          # every ypsend read before the next call overwrites it


def slice_key(evk_full, info, num_q: int):
    """A rank's owned key limbs [dnum][2][nkey][N] from a full key [dnum][2][L+1+K][N]: owned chain
    limbs then owned special limbs (the evk_loc layout of include/hks.h)."""
    import torch
    q = evk_full[:, :, info.q_lo:info.q_hi]
    p = evk_full[:, :, num_q + info.p_lo:num_q + info.p_hi]
    return torch.cat([q, p], dim=2).contiguous()
