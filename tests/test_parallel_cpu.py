"""Multi-GPU host logic on CPU: partitioning and the member-sharded combine,
run with the gloo backend at world size 2 (127.0.0.1 rendezvous)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import cnn
from paper_2008_04063_b200 import arch, parallel
from paper_2008_04063_b200.errors import ConfigurationError
from paper_2008_04063_b200.zoo import Selector, holmes_zoo


def test_patient_shards_are_contiguous_and_balanced():
    for P, W in [(64, 1), (64, 2), (100, 8), (8192, 8), (7, 3)]:
        sh = parallel.patient_shards(P, W)
        assert sh[0][0] == 0 and sum(n for _, n in sh) == P
        assert all(a + n == b for (a, n), (b, _) in zip(sh, sh[1:]))
        assert max(n for _, n in sh) - min(n for _, n in sh) <= 1
    with pytest.raises(ConfigurationError):
        parallel.patient_shards(3, 4)


def test_member_bins_flop_balanced_full_zoo():
    z = holmes_zoo()
    bins = parallel.member_bins(z, Selector.ones(60), 8)
    flat = sorted(i for b in bins for i in b)
    assert flat == list(range(60)) and all(bins)
    loads = [sum(arch.member_flops(z.profiles[i].width, z.profiles[i].depth) for i in b) for b in bins]
    assert max(loads) / min(loads) < 1.25
    assert parallel.member_bins(z, Selector.ones(60), 8) == bins          # deterministic
    with pytest.raises(ConfigurationError):
        parallel.member_bins(z, Selector.from_indices(60, [1, 2]), 3)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, logits, bins, m_total, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = logits[:, bins[rank]].astype(np.float64)
        # what this rank's aggregate kernel writes: fixed-order fp32 partial sums
        sig = np.zeros(logits.shape[0], np.float32)
        lg = np.zeros(logits.shape[0], np.float32)
        for j in range(mine.shape[1]):
            sig += (1.0 / (1.0 + np.exp(-mine[:, j]))).astype(np.float32)
            lg += mine[:, j].astype(np.float32)
        out = parallel.combine_member_sums(torch.from_numpy(np.stack([sig, lg])), m_total)
        if rank == 0:
            q.put((out[0].numpy(), out[1].numpy()))
        else:
            assert out is None
    finally:
        dist.destroy_process_group()


def test_member_sharded_combine_gloo_world2():
    z = holmes_zoo()
    sel = Selector.from_indices(60, [10, 13, 30, 50, 0, 59])
    bins = parallel.member_bins(z, sel, 2)
    order = list(sel.indices())
    rng = np.random.default_rng(0)
    logits = rng.standard_normal((33, 60)).astype(np.float32)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, logits, bins, len(order), q)) for r in range(2)]
    for p in procs:
        p.start()
    prob, lg = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref_prob, ref_logit = cnn.ensemble(logits[:, order])
    assert np.abs(prob - ref_prob).max() < 1e-6 and np.abs(lg - ref_logit).max() < 1e-6


def _gather_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        start, n = parallel.patient_shards(11, world)[rank]

        class R:  # stand-in for this rank's TickResult
            ens_prob = np.arange(start, start + n, dtype=np.float32) / 100
            ens_mean_logit = -np.arange(start, start + n, dtype=np.float32)

        eng = parallel.PatientShardedEngine.__new__(parallel.PatientShardedEngine)
        eng.world = world
        out = eng.gather(R())
        if rank == 0:
            q.put(out)
    finally:
        dist.destroy_process_group()


def test_patient_sharded_gather_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert np.array_equal(out[0], np.arange(11, dtype=np.float32) / 100)
    assert np.array_equal(out[1], -np.arange(11, dtype=np.float32))
