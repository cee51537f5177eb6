"""Multi-GPU serving: one process per GPU, `torch.distributed` for plumbing.

Two ways to spread the tick:

* **Patient sharding** (`PatientShardedEngine`): contiguous bed ranges per
  rank; every rank owns its beds' rings, all selected members' weights and its
  own tick graph.  Beds are independent, so there is NO collective on the data
  path; per-bed results equal the 1-GPU results bit for bit at any shard size
  (every kernel is per bed, and the fused head's partial-sum grouping is fixed
  by the layer shape, not by the batch: `pick_nb` in csrc/conv_pp.cu).  Results are
  gathered to rank 0 only when the caller asks (`gather`).
* **Member sharding** (`MemberShardedEngine`, config c5): the selected members
  are FLOP-balanced over ranks (`member_bins`); every rank ingests every
  stream and runs only its members; its aggregate kernel writes per-bed
  partial sums `[2, P]` (Σ sigmoid, Σ logit, fixed member order) straight into
  a torch-visible device buffer; ONE `reduce(SUM)` to rank 0 per tick (NCCL
  over NVLink on GPUs, 2·P·4 B = 64 KiB at 8192 beds); rank 0's finalize
  kernel divides by the total popcount.  The reference's equivalent is the
  analytic `n_slots` of `ExecutorModel` (`pkg/src/zooserve/latency.py:41-55`).

The partitioning and the combine step are plain functions so the CPU test
suite exercises them with `gloo` at world size 2.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib, arch
from .errors import ConfigurationError
from .zoo import ModelZoo, Selector


def patient_shards(patients: int, world: int) -> list[tuple[int, int]]:
    """Contiguous (start, count) bed ranges, sizes differing by at most one."""
    if world < 1 or patients < world:
        raise ConfigurationError(f"patients: {patients} beds cannot be split over {world} ranks")
    base, extra = divmod(patients, world)
    out, start = [], 0
    for r in range(world):
        n = base + (1 if r < extra else 0)
        out.append((start, n))
        start += n
    return out


def member_bins(zoo: ModelZoo, selector: Selector, world: int) -> list[list[int]]:
    """FLOP-balanced member bins (longest-processing-time greedy; ties -> lower rank).

    Deterministic for a given selector; each bin keeps zoo order; every rank
    gets at least one member.
    """
    idx = list(selector.indices())
    if world < 1 or len(idx) < world:
        raise ConfigurationError(f"selector: {len(idx)} members cannot be split over {world} ranks")
    cost = {i: arch.member_flops(zoo.profiles[i].width, zoo.profiles[i].depth) for i in idx}
    load = [0] * world
    bins: list[list[int]] = [[] for _ in range(world)]
    for i in sorted(idx, key=lambda i: (-cost[i], i)):   # empty ranks (load 0) fill first
        r = min(range(world), key=lambda k: (load[k], k))
        bins[r].append(i)
        load[r] += cost[i]
    return [sorted(b) for b in bins]


class CudaView:
    """Zero-copy `__cuda_array_interface__` over a device pointer (torch.as_tensor wraps it)."""

    def __init__(self, ptr: int, shape, typestr: str = "<f4"):
        self.__cuda_array_interface__ = {"data": (int(ptr), False), "shape": tuple(shape), "typestr": typestr,
                                         "version": 2, "strides": None}


def combine_member_sums(local_sums, m_total: int, group=None, dst: int = 0):
    """SUM-reduce per-rank partial sums [2, P] to `dst`; returns (prob, logit) on dst, else None.

    Works for CUDA tensors (NCCL) and CPU tensors (gloo).  On CUDA the final
    division runs in the library's finalize kernel.
    """
    import torch
    import torch.distributed as dist
    buf = local_sums.clone()
    dist.reduce(buf, dst=dst, op=dist.ReduceOp.SUM, group=group)
    if dist.get_rank(group) != dst:
        return None
    P = buf.shape[1]
    if buf.is_cuda:
        prob = torch.empty(P, dtype=torch.float32, device=buf.device)
        logit = torch.empty_like(prob)
        _lib.check(_lib.lib().hb_finalize_sums(C.c_void_p(buf.data_ptr()), P, int(m_total),
                                               C.c_void_p(prob.data_ptr()), C.c_void_p(logit.data_ptr()),
                                               C.c_void_p(torch.cuda.current_stream().cuda_stream)))
        return prob, logit
    inv = np.float32(1.0) / np.float32(m_total)
    return buf[0] * inv, buf[1] * inv


class PatientShardedEngine:
    """This rank's slice of the beds; no collective per tick."""

    def __init__(self, zoo: ModelZoo, selector: Selector, patients: int, rank: int, world: int, **engine_kw):
        from .engine import EnsembleEngine
        self.rank, self.world = rank, world
        self.start, self.count = patient_shards(patients, world)[rank]
        self.patients = patients
        self.engine = EnsembleEngine(zoo, selector, self.count, **engine_kw)

    def local(self, samples_all: np.ndarray) -> np.ndarray:
        return samples_all[self.start:self.start + self.count]

    def tick(self, samples_local, out=None):
        return self.engine.tick(samples_local, out)

    def gather(self, res, group=None, dst: int = 0):
        """Gather (ens_prob, ens_mean_logit) of every rank's beds to dst in bed order (CPU tensors)."""
        import torch
        import torch.distributed as dist
        loc = torch.from_numpy(np.stack([res.ens_prob, res.ens_mean_logit]).astype(np.float32))
        parts = [None] * self.world if dist.get_rank(group) == dst else None
        dist.gather_object(loc.numpy(), parts, dst=dst, group=group)
        if parts is None:
            return None
        return np.concatenate(parts, axis=1)

    def close(self):
        self.engine.close()


class MemberShardedEngine:
    """This rank's FLOP-balanced share of the members; one SUM reduce per tick.

    Serving path per tick, all stream-ordered on one CUDA stream with a single
    host synchronisation at the end: the hop of every bed is copied into a
    pinned staging buffer and sent H2D in-stream, the tick graph runs this
    rank's members, the per-bed partial sums [2, P] are reduced IN PLACE
    (NCCL over NVLink; the aggregate kernel rewrites them every tick, so no
    copy is needed), and rank 0's finalize kernel divides by the total
    popcount and its D2H lands in pinned host buffers."""

    def __init__(self, zoo: ModelZoo, selector: Selector, patients: int, rank: int, world: int, group=None,
                 **engine_kw):
        import torch

        from .engine import EnsembleEngine
        self.rank, self.world, self.group = rank, world, group
        self.bins = member_bins(zoo, selector, world)
        self.m_total = selector.popcount
        self.patients = patients
        mine = Selector.from_indices(zoo.n, self.bins[rank])
        self.engine = EnsembleEngine(zoo, mine, patients, **engine_kw)
        # a real (non-legacy) stream: the library treats handle 0 as "its own
        # stream", which does not order with torch's legacy default stream
        self.stream = torch.cuda.Stream()
        e = self.engine
        self._stage = torch.empty((patients, e.leads, e.hop), dtype=torch.float32, pin_memory=True)
        self._stage_np = self._stage.numpy()
        self._prob = torch.empty(patients, dtype=torch.float32, device="cuda")
        self._logit = torch.empty(patients, dtype=torch.float32, device="cuda")
        self._h_out = torch.empty((2, patients), dtype=torch.float32, pin_memory=True)
        self._sums = None

    def _sums_tensor(self):
        import torch
        ptr = C.c_void_p()   # (valid once a tick built the selection; re-read: a rebuild moves it)
        _lib.check(_lib.lib().hb_device_sums(self.engine._h, C.byref(ptr)), self.engine._h)
        if self._sums is None or self._sums.data_ptr() != ptr.value:
            self._sums = torch.as_tensor(CudaView(ptr.value, (2, self.patients)), device="cuda")
        return self._sums

    def reduce_device(self, stream=None) -> None:
        """After this rank's tick on `stream`: the in-place NCCL reduce of the partial sums to rank 0 and
        (rank 0) the finalize kernel into device buffers; stream-ordered, no host synchronisation."""
        import torch
        import torch.distributed as dist
        stream = stream or self.stream
        with torch.cuda.stream(stream):
            sums = self._sums_tensor()
            dist.reduce(sums, dst=0, op=dist.ReduceOp.SUM, group=self.group)
            if dist.get_rank(self.group) == 0:
                _lib.check(_lib.lib().hb_finalize_sums(C.c_void_p(sums.data_ptr()), self.patients, int(self.m_total),
                                                       C.c_void_p(self._prob.data_ptr()),
                                                       C.c_void_p(self._logit.data_ptr()),
                                                       C.c_void_p(stream.cuda_stream)))

    def finished_outputs(self):
        """(prob, mean_logit) numpy of the last reduced tick on rank 0 (synchronises), else (None, None)."""
        import torch.distributed as dist
        self.stream.synchronize()
        import torch
        torch.cuda.synchronize()
        if dist.get_rank(self.group) != 0:
            return None, None
        return self._prob.cpu().numpy(), self._logit.cpu().numpy()

    def tick(self, samples_all: np.ndarray):
        """Every rank passes ALL beds' samples [P, leads, hop]; rank 0 gets (prob, mean_logit) as CPU tensors,
        the other ranks None."""
        import torch
        import torch.distributed as dist
        e = self.engine
        np.copyto(self._stage_np, samples_all, casting="same_kind")
        st = self.stream
        with e._lock:
            rc = _lib.lib().hb_tick(e._h, C.c_void_p(self._stage_np.ctypes.data), None, None, None,
                                    C.c_void_p(st.cuda_stream))
        if rc:
            _lib.check(rc, e._h)
        self.reduce_device(st)
        root = dist.get_rank(self.group) == 0
        if root:
            with torch.cuda.stream(st):
                self._h_out[0].copy_(self._prob, non_blocking=True)
                self._h_out[1].copy_(self._logit, non_blocking=True)
        st.synchronize()
        return (self._h_out[0].clone(), self._h_out[1].clone()) if root else None

    def close(self):
        self._sums = None
        self.engine.close()
