"""Multi-rank runs of bench.py checked against the CPU oracle.

On the one-GPU box both ranks share cuda:0 and talk over gloo (HKS_BENCH_BACKEND=gloo): the timings of such
a run mean nothing, but every rank runs the code path of the multi-GPU bench -- the C3 ciphertext sharding
and the C4 limb sharding with its two all-gathers issued by paper_2507_04775_b200.shard -- and dumps one
step's inputs and outputs (`--dump`).  The test reassembles them and compares with the oracle bit for bit:
C4 = oracle KeySwitch of the full ciphertext with the full key (the union of the ranks' limb slices), C3 =
oracle hoisted rotations of each rank's first ciphertext."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import hks_synth as S

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(tmp_path, args, world=2):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    d = str(tmp_path / "dump")
    port = 29400 + os.getpid() % 500
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.join(ROOT, "bench.py"),
           "--gpus", str(world), "--steps", "2", "--warmup", "3", "--quick", "--dump", d] + args
    r = subprocess.run(cmd, cwd=ROOT, env=dict(os.environ, HKS_BENCH_BACKEND="gloo"), capture_output=True,
                       text=True, timeout=1500)
    assert r.returncode == 0, (r.stdout[-3000:], r.stderr[-3000:])
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]               # one JSON line, from rank 0
    line = json.loads(lines[0])
    assert line["n_gpus"] == world and line["value"] > 0
    return d, line


def _load(d, rank):
    p = os.path.join(d, f"rank{rank}")
    with open(os.path.join(p, "meta.json")) as f:
        meta = json.load(f)
    arr = {k[:-4]: np.load(os.path.join(p, k)) for k in os.listdir(p) if k.endswith(".npy")}
    return meta, arr


def test_c4_limb_sharded_two_ranks(orc, tmp_path):
    """C4 (BASELINE configs[3]) limb-sharded over two ranks, NCCL-mode exchange (all_gather_into_tensor, here
    over gloo): the ranks' output slices together equal the oracle KeySwitch of the assembled inputs."""
    d, line = _run(tmp_path, ["--config", "C4", "--shard", "nccl", "--sets", "1"])
    assert "RNS limbs sharded over 2" in line["config"]["parallelism"]
    cfg = S.config("C4")
    o = orc.Ctx.from_config(cfg)
    nq, nk = len(cfg.q), len(cfg.q) + len(cfg.p)
    parts = [_load(d, r) for r in range(2)]
    level = parts[0][0]["level"]
    c0 = np.concatenate([a["c0"] for m, a in parts])
    c1 = np.concatenate([a["c1"] for m, a in parts])
    got0 = np.concatenate([a["out0"] for m, a in parts])
    got1 = np.concatenate([a["out1"] for m, a in parts])
    evk = np.zeros((cfg.dnum, 2, nk, o.n), dtype=np.uint64)
    for m, a in parts:
        nql = m["q_hi"] - m["q_lo"]
        evk[:, :, m["q_lo"]:m["q_hi"]] = a["evk"][:, :, :nql]
        evk[:, :, nq + m["p_lo"]:nq + m["p_hi"]] = a["evk"][:, :, nql:]
    assert c0.shape[0] == level + 1
    want0, want1 = o.keyswitch(c0, c1, evk, level)
    assert (got0 == want0).all() and (got1 == want1).all()


def test_c3_ciphertext_sharded_two_ranks(orc, tmp_path):
    """C3 (BASELINE configs[2]) with its 8 ciphertexts sharded over two ranks: each rank's hoisted rotations
    (first and last rotation of its first ciphertext) equal the oracle's."""
    d, line = _run(tmp_path, ["--config", "C3"])
    cfg = S.config("C3")
    o = orc.Ctx.from_config(cfg)
    for r in range(2):
        m, a = _load(d, r)
        outs0, outs1 = o.rotate_hoisted(a["c0"], a["c1"], [a["evk"][k] for k in range(2)], m["level"], m["galois"])
        for k in range(2):
            assert (a["out0"][k] == outs0[k]).all() and (a["out1"][k] == outs1[k]).all(), (r, k)


@pytest.mark.parametrize("mode,tag", [("pipe", "per-digit broadcasts"), ("a2a", "four all-to-alls")])
def test_c4_exchange_variants_two_ranks(orc, tmp_path, mode, tag):
    """C4 limb-sharded with the NEXT-3 exchange variants, two ranks: the first exchange as per-digit broadcasts
    pipelined with the conversions (pipe), or coefficient-sharded conversions with four all-to-alls (a2a);
    bit-exact with the oracle."""
    d, line = _run(tmp_path, ["--config", "C4", "--shard", mode, "--sets", "1"])
    assert tag in line["config"]["l2"]
    cfg = S.config("C4")
    o = orc.Ctx.from_config(cfg)
    nq, nk = len(cfg.q), len(cfg.q) + len(cfg.p)
    parts = [_load(d, r) for r in range(2)]
    level = parts[0][0]["level"]
    c0 = np.concatenate([a["c0"] for m, a in parts])
    c1 = np.concatenate([a["c1"] for m, a in parts])
    got0 = np.concatenate([a["out0"] for m, a in parts])
    got1 = np.concatenate([a["out1"] for m, a in parts])
    evk = np.zeros((cfg.dnum, 2, nk, o.n), dtype=np.uint64)
    for m, a in parts:
        nql = m["q_hi"] - m["q_lo"]
        evk[:, :, m["q_lo"]:m["q_hi"]] = a["evk"][:, :, :nql]
        evk[:, :, nq + m["p_lo"]:nq + m["p_hi"]] = a["evk"][:, :, nql:]
    want0, want1 = o.keyswitch(c0, c1, evk, level)
    assert (got0 == want0).all() and (got1 == want1).all()
