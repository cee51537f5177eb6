"""Multi-GPU paths on one B200: member-sharded partial sums + finalize kernel
(two contexts on one device stand in for two ranks), the NCCL reduce with a
world-size-1 group, and patient sharding's bit-identity with 1 GPU."""
import os
import socket

import numpy as np
import pytest
import torch

from paper_2008_04063_b200 import parallel, synth
from paper_2008_04063_b200.engine import EnsembleEngine
from paper_2008_04063_b200.zoo import Selector, holmes_zoo

pytestmark = pytest.mark.gpu
SEL = [0, 10, 13, 21, 30, 50]


def _streams(P, n=7500, seed=2):
    return synth.ecg_block(seed, P, 3, 0, n)


def test_member_shards_sum_to_the_full_ensemble():
    zoo = holmes_zoo()
    sel = Selector.from_indices(60, SEL)
    P = 5
    s = _streams(P)
    with EnsembleEngine(zoo, sel, P) as full:
        ref = full.tick(s)
    bins = parallel.member_bins(zoo, sel, 2)
    sums = torch.zeros(2, P, device="cuda")
    engines = []
    try:
        for b in bins:
            e = EnsembleEngine(zoo, Selector.from_indices(60, b), P)
            engines.append(e)
            e.tick(s)
            import ctypes as C
            from paper_2008_04063_b200 import _lib
            ptr = C.c_void_p()
            _lib.check(_lib.lib().hb_device_sums(e._h, C.byref(ptr)))
            sums += torch.as_tensor(parallel.CudaView(ptr.value, (2, P)), device="cuda")
    finally:
        for e in engines:
            e.close()
    prob = torch.empty(P, device="cuda")
    logit = torch.empty(P, device="cuda")
    import ctypes as C
    from paper_2008_04063_b200 import _lib
    _lib.check(_lib.lib().hb_finalize_sums(C.c_void_p(sums.data_ptr()), P, len(SEL), C.c_void_p(prob.data_ptr()),
                                           C.c_void_p(logit.data_ptr()), None))
    torch.cuda.synchronize()
    assert np.abs(prob.cpu().numpy() - ref.ens_prob).max() < 1e-5
    assert np.abs(logit.cpu().numpy() - ref.ens_mean_logit).max() < 1e-4


def test_member_sharded_engine_nccl_world1():
    import torch.distributed as dist
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        zoo = holmes_zoo()
        sel = Selector.from_indices(60, SEL)
        P, hop = 4, 7500
        s = _streams(P)
        me = parallel.MemberShardedEngine(zoo, sel, P, 0, 1, hop=hop)
        try:
            prob, logit = me.tick(s)
        finally:
            me.close()
        with EnsembleEngine(zoo, sel, P, hop=hop) as full:
            ref = full.tick(s)
        assert np.abs(prob.cpu().numpy() - ref.ens_prob).max() < 1e-6
        assert np.abs(logit.cpu().numpy() - ref.ens_mean_logit).max() < 1e-6
    finally:
        dist.destroy_process_group()


def test_patient_shards_bit_identical_to_one_gpu():
    zoo = holmes_zoo()
    sel = Selector.from_indices(60, [10, 13])
    P = 7
    s = _streams(P, seed=5)
    with EnsembleEngine(zoo, sel, P) as full:
        ref = full.tick(s)
    for rank in range(3):
        start, n = parallel.patient_shards(P, 3)[rank]
        with EnsembleEngine(zoo, sel, n) as e:
            r = e.tick(s[start:start + n])
        assert np.array_equal(r.member_logits, ref.member_logits[start:start + n])
        assert np.array_equal(r.ens_prob, ref.ens_prob[start:start + n])
