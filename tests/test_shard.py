"""Limb-sharded KeySwitch.

CPU (gloo, world_size 2): the ownership plan is a partition, and the all-gather layout the Python
orchestrator produces matches the slots libhks reads (q_slot / p_slot).
GPU: G simulated ranks on one device (all-gather = local concatenation) give results bit-identical to the
CPU oracle's KeySwitch on the same inputs (and hence to the unsharded hks_keyswitch; integer math is
order-independent: SURVEY.md §4 item 5, "sharded == unsharded" anchored on the oracle, SURVEY.md:703)."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import hks_synth as S

H = pytest.importorskip("paper_2507_04775_b200.hks")
from paper_2507_04775_b200 import shard  # noqa: E402


@pytest.mark.parametrize("name,level", [("C4", 35), ("C4", 20), ("C2", 29), ("T12", 6), ("T12", 2)])
def test_plan_is_partition(name, level):
    cfg = S.config(name)
    ctx = H.Context.from_config(cfg, -1)
    for world in (1, 2, 3, 4, 8):
        if world > len(cfg.q):
            continue
        infos = [H.shard_query(ctx, level, world, r) for r in range(world)]
        q_owned = [i for s in infos for i in range(s.q_lo, s.q_hi)]
        p_owned = [k for s in infos for k in range(s.p_lo, s.p_hi)]
        assert q_owned == list(range(len(cfg.q))) and p_owned == list(range(len(cfg.p)))
        tot = [(s.q_hi - s.q_lo) + (s.p_hi - s.p_lo) for s in infos]
        assert max(tot) - min(tot) <= 2
        assert sum(s.nq_act for s in infos) == level + 1
        assert all(s.q_pad == max(x.q_hi - x.q_lo for x in infos) for s in infos)


def _gloo_worker(rank, world, port, name, level, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = S.config(name)
        ctx = H.Context.from_config(cfg, -1)
        plan = shard.ShardPlan(ctx, level, world)
        me = plan.info[rank]
        n = 8                                               # stand-in row length
        ysend = torch.full((me.q_pad, n), -1, dtype=torch.int64)
        for li in range(me.nq_act):
            ysend[li] = me.q_lo + li                        # marker: global chain limb index
        ypsend = torch.full((2 * me.p_pad, n), -1, dtype=torch.int64)
        for poly in range(2):
            for kk in range(me.p_hi - me.p_lo):
                ypsend[poly * me.p_pad + kk] = 1000 * (poly + 1) + me.p_lo + kk
        yall = torch.empty((world * me.q_pad, n), dtype=torch.int64)
        ypall = torch.empty((world * 2 * me.p_pad, n), dtype=torch.int64)
        dist.all_gather_into_tensor(yall, ysend)
        dist.all_gather_into_tensor(ypall, ypsend)
        ok = all(int(yall[plan.q_slot(i), 0]) == i for i in range(level + 1))
        ok &= all(int(ypall[plan.p_slot(k, poly), 0]) == 1000 * (poly + 1) + k
                  for k in range(len(cfg.p)) for poly in range(2))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,level", [("C4", 35), ("T12", 5)])
def test_gloo_allgather_layout(name, level):
    world = 2
    ctxmp = mp.get_context("spawn")
    q = ctxmp.Queue()
    port = 29500 + (os.getpid() % 1000)
    procs = [ctxmp.Process(target=_gloo_worker, args=(r, world, port, name, level, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok in res), res


def _gloo_pipe_worker(rank, world, port, name, level, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = S.config(name)
        ctx = H.Context.from_config(cfg, -1)
        plan = shard.ShardPlan(ctx, level, world)
        me = plan.info[rank]
        segs = shard.digit_segments(ctx, level, world)
        n = 4
        yall = torch.full((world * me.q_pad, n), -1, dtype=torch.int64)
        for li in range(me.nq_act):
            yall[rank * me.q_pad + li] = me.q_lo + li           # own slots = phase A output (marker: limb index)
        for runs in segs:                                       # one broadcast per (digit, owner) run
            for r, lo, hi in runs:
                dist.broadcast(yall[lo:hi], src=r)
        ok = all(int(yall[plan.q_slot(i), 0]) == i for i in range(level + 1))
        info = ctx.query(level)
        for j, runs in enumerate(segs):                         # the runs of digit j are exactly its limbs
            got = sorted(int(yall[s_, 0]) for _, lo, hi in runs for s_ in range(lo, hi))
            ok &= got == list(range(info.digit_lo[j], info.digit_hi[j]))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,level,world", [("C4", 35, 2), ("C4", 20, 2), ("T12", 5, 2)])
def test_gloo_digit_broadcast_layout(name, level, world):
    """NEXT-3 pipelined exchange: per-digit broadcasts of the owners' runs fill the gathered buffer exactly as
    the all-gather does, and each digit's runs cover that digit's limbs."""
    ctxmp = mp.get_context("spawn")
    q = ctxmp.Queue()
    port = 29700 + (os.getpid() % 1000)
    procs = [ctxmp.Process(target=_gloo_pipe_worker, args=(r, world, port, name, level, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok in res), res


def _gloo_a2a_worker(rank, world, port, name, level, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = S.config(name)
        ctx = H.Context.from_config(cfg, -1)
        infos = [H.shard_query(ctx, level, world, r) for r in range(world)]
        me = infos[rank]
        nc = H.shard_a2a_query(ctx, level, world, rank).chunk_words
        assert nc * world == cfg.n
        # chunked send buffer [G][q_pad][Nc]: chunk k of own limb li carries (limb index, chunk k)
        ysend = torch.full((world * me.q_pad, 2), -1, dtype=torch.int64)
        for k in range(world):
            for li in range(me.nq_act):
                ysend[k * me.q_pad + li] = torch.tensor([me.q_lo + li, k])
        yrecv = torch.empty_like(ysend)
        dist.all_to_all_single(yrecv, ysend)
        # after the exchange: slot r * q_pad + (i - q_lo(r)) holds chain limb i, this rank's chunk
        ok = True
        for i in range(level + 1):
            r = next(r for r, s_ in enumerate(infos) if s_.q_lo <= i < s_.q_hi)
            ok &= yrecv[r * me.q_pad + i - infos[r].q_lo].tolist() == [i, rank]
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,level,world", [("C4", 35, 2), ("C4", 17, 2), ("T12", 6, 2)])
def test_gloo_a2a_chunk_layout(name, level, world):
    """NEXT-3 coefficient-sharded exchange: all_to_all_single of the chunked send buffers gives every rank its
    chunk of every active chain limb at the all-gather slot positions (include/hks.h, phase 1 -> 2)."""
    ctxmp = mp.get_context("spawn")
    q = ctxmp.Queue()
    port = 29900 + (os.getpid() % 1000)
    procs = [ctxmp.Process(target=_gloo_a2a_worker, args=(r, world, port, name, level, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok in res), res


# ------------------------------------------------------------------ GPU: simulated ranks
def _oracle_ks(orc, cfg, c0, c1, evk, level):
    """the CPU oracle's KeySwitch on the device inputs (uint64 views)"""
    o = orc.Ctx.from_config(cfg)
    h = lambda t: t.cpu().numpy().view(np.uint64)
    return o.keyswitch(h(c0), h(c1), h(evk), level)


def _equal_oracle(got0, got1, want):
    h = lambda t: t.cpu().numpy().view(np.uint64)
    return bool((h(got0) == want[0]).all() and (h(got1) == want[1]).all())


@pytest.mark.gpu
@pytest.mark.parametrize("name,level,world", [("T12", 6, 2), ("T12", 4, 3), ("T16s", 5, 2), ("C2", 29, 4),
                                              ("C4", 35, 8), ("C4", 35, 2), ("C4", 17, 4)])
def test_sharded_keyswitch_matches_unsharded(orc, name, level, world):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    dev = "cuda:0"
    cfg = S.config(name)
    ctx = H.Context.from_config(cfg, 0)
    g = torch.Generator(device=dev)
    g.manual_seed(cfg.seed)
    n = cfg.n
    primes = list(cfg.q) + list(cfg.p)

    def limbs(pr):
        return torch.stack([torch.randint(0, int(p), (n,), generator=g, device=dev, dtype=torch.int64) for p in pr])

    c0, c1 = limbs(cfg.q[: level + 1]), limbs(cfg.q[: level + 1])
    evk = torch.stack([limbs(primes) for _ in range(2 * cfg.dnum)]).reshape(cfg.dnum, 2, len(primes), n)
    ref0, ref1 = torch.empty_like(c0), torch.empty_like(c1)
    H.keyswitch(ctx, c0, c1, level, evk, ref0, ref1, ctx.workspace(H.OP_KEYSWITCH, level))

    ranks = [shard.ShardedKeySwitch(ctx, level, world, r, dev, gather_fn=lambda o, i: None) for r in range(world)]
    loc = []
    for r, ks in enumerate(ranks):
        s = ks.info
        c0l, c1l = c0[s.q_lo:s.q_lo + s.nq_act].contiguous(), c1[s.q_lo:s.q_lo + s.nq_act].contiguous()
        loc.append((c0l, c1l, shard.slice_key(evk, s, len(cfg.q)), torch.empty_like(c0l), torch.empty_like(c1l)))
        ks.phase_a(c1l)
    yall = torch.cat([ks.ysend for ks in ranks])
    for r, ks in enumerate(ranks):
        ks.yall.copy_(yall)
        ks.phase_b(loc[r][1], loc[r][2])
    ypall = torch.cat([ks.ypsend for ks in ranks])
    for r, ks in enumerate(ranks):
        ks.ypall.copy_(ypall)
        c0l, c1l, _, o0, o1 = loc[r]
        ks.phase_c(c0l, o0, o1)
    got0 = torch.cat([l[3] for l in loc])
    got1 = torch.cat([l[4] for l in loc])
    torch.cuda.synchronize()
    assert _equal_oracle(got0, got1, _oracle_ks(orc, cfg, c0, c1, evk, level))
    assert torch.equal(got0, ref0) and torch.equal(got1, ref1)


@pytest.mark.gpu
@pytest.mark.parametrize("name,level,world", [("T12", 6, 2), ("T12", 4, 3), ("C2", 29, 4), ("C4", 35, 8),
                                              ("C4", 35, 2), ("C4", 17, 4)])
def test_peer_sharded_keyswitch_matches_unsharded(orc, name, level, world):
    """NEXT-3: phases B and C read the other ranks' limbs through a pointer table (here: simulated ranks'
    buffers on one GPU) inside the base conversion; bit-identical to hks_keyswitch."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    dev = "cuda:0"
    cfg = S.config(name)
    ctx = H.Context.from_config(cfg, 0)
    g = torch.Generator(device=dev)
    g.manual_seed(cfg.seed + 1)
    n = cfg.n
    primes = list(cfg.q) + list(cfg.p)

    def limbs(pr):
        return torch.stack([torch.randint(0, int(p), (n,), generator=g, device=dev, dtype=torch.int64) for p in pr])

    c0, c1 = limbs(cfg.q[: level + 1]), limbs(cfg.q[: level + 1])
    evk = torch.stack([limbs(primes) for _ in range(2 * cfg.dnum)]).reshape(cfg.dnum, 2, len(primes), n)
    ref0, ref1 = torch.empty_like(c0), torch.empty_like(c1)
    H.keyswitch(ctx, c0, c1, level, evk, ref0, ref1, ctx.workspace(H.OP_KEYSWITCH, level))

    infos = [H.shard_query(ctx, level, world, r) for r in range(world)]
    ys = [torch.full((s.q_pad, n), -1, dtype=torch.int64, device=dev) for s in infos]
    yps = [torch.full((2 * s.p_pad, n), -1, dtype=torch.int64, device=dev) for s in infos]
    ranks = [shard.PeerShardedKeySwitch(ctx, level, world, r, dev, sim_ysend=ys, sim_ypsend=yps)
             for r in range(world)]
    loc = []
    for ks in ranks:
        s = ks.info
        c0l, c1l = c0[s.q_lo:s.q_lo + s.nq_act].contiguous(), c1[s.q_lo:s.q_lo + s.nq_act].contiguous()
        loc.append((c0l, c1l, shard.slice_key(evk, s, len(cfg.q)), torch.empty_like(c0l), torch.empty_like(c1l)))
        ks.phase_a(c1l)
    for r, ks in enumerate(ranks):
        ks.phase_b(loc[r][1], loc[r][2])
    for r, ks in enumerate(ranks):
        c0l, _, _, o0, o1 = loc[r]
        ks.phase_c(c0l, o0, o1)
    torch.cuda.synchronize()
    got0, got1 = torch.cat([l[3] for l in loc]), torch.cat([l[4] for l in loc])
    assert _equal_oracle(got0, got1, _oracle_ks(orc, cfg, c0, c1, evk, level))
    assert torch.equal(got0, ref0) and torch.equal(got1, ref1)


@pytest.mark.gpu
def test_peer_phase_rejects_null_table():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cfg = S.config("T12")
    ctx = H.Context.from_config(cfg, 0)
    s = H.shard_query(ctx, 4, 2, 0)
    z = torch.zeros((8, cfg.n), dtype=torch.int64, device="cuda:0")
    with pytest.raises(H.HksError):
        H.shard_ks_inner_peer(ctx, 4, 2, 0, [z.data_ptr(), 0], z, z, z, z, z)


@pytest.mark.gpu
@pytest.mark.parametrize("name,level,world", [("T12", 6, 2), ("T12", 4, 3), ("C2", 29, 4), ("C4", 35, 8), ("C4", 35, 2),
                                              ("C4", 17, 4)])
def test_pipelined_sharded_keyswitch_matches_oracle(orc, name, level, world):
    """NEXT-3 per-digit pipelined first exchange: each simulated rank receives digit j by copies of the owners'
    runs on an auxiliary stream, recorded by an event that phase B waits on before digit j's conversion; the
    outputs equal the CPU oracle's KeySwitch."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    dev = "cuda:0"
    cfg = S.config(name)
    ctx = H.Context.from_config(cfg, 0)
    g = torch.Generator(device=dev)
    g.manual_seed(cfg.seed + 2)
    n = cfg.n
    primes = list(cfg.q) + list(cfg.p)

    def limbs(pr):
        return torch.stack([torch.randint(0, int(p), (n,), generator=g, device=dev, dtype=torch.int64) for p in pr])

    c0, c1 = limbs(cfg.q[: level + 1]), limbs(cfg.q[: level + 1])
    evk = torch.stack([limbs(primes) for _ in range(2 * cfg.dnum)]).reshape(cfg.dnum, 2, len(primes), n)
    ranks = []

    def deliver_for(me):
        def deliver(j, runs, yall):
            for r, lo, hi in runs:
                if r != me:
                    yall[lo:hi].copy_(ranks[r].yall[lo:hi])
        return deliver

    ranks.extend(shard.PipelinedShardedKeySwitch(ctx, level, world, r, dev, deliver_fn=deliver_for(r),
                                                 gather_fn=lambda o, i: None) for r in range(world))
    loc = []
    for ks in ranks:
        s = ks.info
        c0l, c1l = c0[s.q_lo:s.q_lo + s.nq_act].contiguous(), c1[s.q_lo:s.q_lo + s.nq_act].contiguous()
        loc.append((c0l, c1l, shard.slice_key(evk, s, len(cfg.q)), torch.empty_like(c0l), torch.empty_like(c1l)))
        ks.phase_a(c1l)
    for r, ks in enumerate(ranks):
        ks.deliver_digits()
        ks.phase_b(loc[r][1], loc[r][2])
    ypall = torch.cat([ks.ypsend for ks in ranks])
    for r, ks in enumerate(ranks):
        ks.ypall.copy_(ypall)
        c0l, _, _, o0, o1 = loc[r]
        ks.phase_c(c0l, o0, o1)
    torch.cuda.synchronize()
    got0, got1 = torch.cat([l[3] for l in loc]), torch.cat([l[4] for l in loc])
    assert _equal_oracle(got0, got1, _oracle_ks(orc, cfg, c0, c1, evk, level))


@pytest.mark.gpu
@pytest.mark.parametrize("name,level,world", [("T12", 6, 2), ("T12", 4, 4), ("C2", 29, 4), ("C2", 12, 2), ("C4", 35, 8),
                                              ("C4", 35, 2), ("C4", 17, 4)])
def test_a2a_sharded_keyswitch_matches_oracle(orc, name, level, world):
    """NEXT-3 coefficient-sharded base conversions: four all-to-alls (simulated between ranks on one GPU:
    part k of rank r's send buffer -> part r of rank k's receive buffer); the outputs equal the oracle's."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    dev = "cuda:0"
    cfg = S.config(name)
    ctx = H.Context.from_config(cfg, 0)
    g = torch.Generator(device=dev)
    g.manual_seed(cfg.seed + 3)
    n = cfg.n
    primes = list(cfg.q) + list(cfg.p)

    def limbs(pr):
        return torch.stack([torch.randint(0, int(p), (n,), generator=g, device=dev, dtype=torch.int64) for p in pr])

    c0, c1 = limbs(cfg.q[: level + 1]), limbs(cfg.q[: level + 1])
    evk = torch.stack([limbs(primes) for _ in range(2 * cfg.dnum)]).reshape(cfg.dnum, 2, len(primes), n)
    ranks = [shard.A2AShardedKeySwitch(ctx, level, world, r, dev, a2a_fn=lambda o, i: None) for r in range(world)]

    def exchange(name_s, name_r):
        sends = [getattr(k, name_s) for k in ranks]
        for kk, k in enumerate(ranks):
            recv = getattr(k, name_r)
            part = recv.shape[0] // world
            for r in range(world):
                recv[r * part:(r + 1) * part].copy_(sends[r][kk * part:(kk + 1) * part])

    loc = []
    for ks in ranks:
        s = ks.info
        c0l, c1l = c0[s.q_lo:s.q_lo + s.nq_act].contiguous(), c1[s.q_lo:s.q_lo + s.nq_act].contiguous()
        loc.append((c0l, c1l, shard.slice_key(evk, s, len(cfg.q)), torch.empty_like(c0l), torch.empty_like(c1l)))
        ks.phase1(c1l)
    exchange("ysend", "yrecv")
    for ks in ranks:
        ks.phase2()
    exchange("extsend", "extrecv")
    for r, ks in enumerate(ranks):
        ks.phase3(loc[r][1], loc[r][2])
    exchange("ypsend", "yprecv")
    for ks in ranks:
        ks.phase4()
    exchange("convsend", "convrecv")
    for r, ks in enumerate(ranks):
        c0l, _, _, o0, o1 = loc[r]
        ks.phase5(c0l, o0, o1)
    torch.cuda.synchronize()
    got0, got1 = torch.cat([l[3] for l in loc]), torch.cat([l[4] for l in loc])
    assert _equal_oracle(got0, got1, _oracle_ks(orc, cfg, c0, c1, evk, level))
