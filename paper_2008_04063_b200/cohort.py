"""Labelled cohorts and the accuracy profiler f_a, backed by the K6 sweep kernel.

Drop-in for `pkg/src/zooserve/cohort.py`:

* `positive_shift`, `Cohort`, `synthesize_cohort` (the reference's binormal
  cohort, bit-identical per seed — pinned by tests/golden/cohort.json),
  `ensemble_scores`, `ensemble_roc_auc`, `accuracy_profile`
  (`cohort.py:27-115`).  The ensemble means and every ROC-AUC are computed on
  the device (`hb_cohort_*`, csrc/sweep.cu).
* `record_cohort` is what the north star adds: every zoo member's real
  forward over recorded windows (the serving kernels, `engine.py`) fills
  `Cohort.scores` with member logits, so the profiler sweep runs on the same
  kernels that serve.

`DeviceCohort` is the device-resident form (scores uploaded once, column-major,
smaller class first); a `Cohort` caches one per device.
"""

from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass
from statistics import NormalDist

import numpy as np

from . import _lib
from .errors import EmptyEnsembleError
from .zoo import ModelZoo, Selector

_NORMAL = NormalDist()


def positive_shift(target_auc: float) -> float:
    """Binormal separation mu = sqrt(2) * Phi^-1(auc) that realises `target_auc`."""
    return float(np.sqrt(2.0) * _NORMAL.inv_cdf(target_auc))


class DeviceCohort:
    """scores [N, n] fp64 + labels [N] resident on one GPU (hb_cohort)."""

    def __init__(self, scores: np.ndarray, labels: np.ndarray, device: int = 0):
        sc = np.ascontiguousarray(scores, dtype=np.float64)
        lab = np.ascontiguousarray(labels, dtype=np.int8)
        if sc.ndim != 2 or lab.ndim != 1 or sc.shape[0] != lab.size:
            raise ValueError("labels must be 1-D and scores (n_samples, n_models)")
        self.N, self.n = sc.shape
        L = _lib.lib()
        h = C.c_void_p()
        _lib.check(L.hb_cohort_create(device, _lib.dptr(sc), lab.ctypes.data_as(C.POINTER(C.c_int8)), self.N,
                                      self.n, C.byref(h)), None, "hb_cohort_last_error")
        self._h = h
        self._lock = threading.Lock()

    def _check(self, rc: int) -> None:
        _lib.check(rc, self._h, "hb_cohort_last_error")

    def auc_bits(self, bits: np.ndarray) -> np.ndarray:
        """AUC of the mean of every selector row bits[S, n] (0/1)."""
        b = np.ascontiguousarray(bits, dtype=np.uint8)
        if b.ndim != 2 or b.shape[1] != self.n:
            raise ValueError(f"selector rows must have length {self.n}")
        out = np.empty(b.shape[0])
        with self._lock:
            self._check(_lib.lib().hb_cohort_auc(self._h, b.ctypes.data_as(C.POINTER(C.c_uint8)), b.shape[0],
                                                 _lib.dptr(out)))
        return out

    def auc_range(self, first: int, count: int) -> np.ndarray:
        """AUC of the candidates with integer values first .. first+count-1 (bit k <-> column k)."""
        out = np.empty(int(count))
        with self._lock:
            self._check(_lib.lib().hb_cohort_auc_range(self._h, int(first), int(count), _lib.dptr(out)))
        return out

    def ensemble(self, bits) -> tuple[np.ndarray, float]:
        """(ensemble means [N] in row order, their AUC) of one selector."""
        b = np.ascontiguousarray(bits, dtype=np.uint8)
        ens = np.empty(self.N)
        auc = C.c_double()
        with self._lock:
            self._check(_lib.lib().hb_cohort_ensemble(self._h, b.ctypes.data_as(C.POINTER(C.c_uint8)),
                                                      _lib.dptr(ens), C.byref(auc)))
        return ens, auc.value

    def close(self) -> None:
        if getattr(self, "_h", None):
            _lib.lib().hb_cohort_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass(frozen=True)
class Cohort:
    """Labels int8[N] (both classes) plus one finite fp64 score column per zoo member.

    Same invariants as the reference (`cohort.py:32-56`); arrays are frozen
    read-only.  The device copy is built lazily, once per GPU.
    """

    labels: np.ndarray
    scores: np.ndarray
    seed: int

    def __post_init__(self):
        lab = np.array(self.labels, dtype=np.int8)
        sc = np.array(self.scores, dtype=np.float64)
        if lab.ndim != 1 or sc.ndim != 2 or sc.shape[0] != lab.size:
            raise ValueError("labels must be 1-D and scores (n_samples, n_models)")
        if lab.min() == lab.max():
            raise ValueError("cohort needs both classes present")
        if not np.isfinite(sc).all():
            raise ValueError("scores must be finite")
        for a in (lab, sc):
            a.setflags(write=False)
        object.__setattr__(self, "labels", lab)
        object.__setattr__(self, "scores", sc)
        object.__setattr__(self, "_dev", {})

    @property
    def n_models(self) -> int:
        return self.scores.shape[1]

    def device(self, device: int = 0) -> DeviceCohort:
        dev = self._dev.get(device)
        if dev is None:
            dev = DeviceCohort(self.scores, self.labels, device)
            self._dev[device] = dev
        return dev

    def __hash__(self):
        return id(self)

    def __eq__(self, other):
        return self is other


@dataclass(frozen=True)
class AccuracyReport:
    roc_auc: float
    pr_auc: float
    f1: float
    accuracy: float


def synthesize_cohort(zoo: ModelZoo, n_pos: int, n_neg: int, correlation: float = 0.5, seed: int = 0) -> Cohort:
    """The reference's binormal cohort (`cohort.py:67-86`), same RNG stream per seed:
    score_j = mu_j * label + sqrt(rho) * shared + sqrt(1 - rho) * private_j."""
    if n_pos < 1 or n_neg < 1:
        raise ValueError("n_pos and n_neg must be >= 1")
    if not 0.0 <= correlation < 1.0:
        raise ValueError("correlation must lie in [0, 1)")
    mu = np.array([positive_shift(p.target_auc) for p in zoo.profiles])
    rng = np.random.default_rng(seed)
    N = n_pos + n_neg
    labels = np.r_[np.ones(n_pos, np.int8), np.zeros(n_neg, np.int8)]
    shared = rng.standard_normal((N, 1))
    private = rng.standard_normal((N, zoo.n))
    scores = mu[None, :] * labels[:, None] + np.sqrt(correlation) * shared + np.sqrt(1.0 - correlation) * private
    return Cohort(labels=labels, scores=scores, seed=seed)


def _bits(cohort: Cohort, b: Selector) -> np.ndarray:
    if b.n != cohort.n_models:
        raise ValueError(f"selector length {b.n} does not match cohort width {cohort.n_models}")
    if b.popcount == 0:
        raise EmptyEnsembleError("cannot score an empty ensemble")
    return np.array(b.bits, dtype=np.uint8)


MAX_DEVICE_COLUMNS = 256   # the K6 kernel's column list (csrc/sweep.cu kMaxCols)


def _device_and_bits(cohort: Cohort, b: Selector, device: int):
    """The device cohort and selector bits to score b with.  Cohorts wider than the kernel's column
    list (the reference accepts any width) are scored on a device sub-cohort of just the selected
    columns, in column order (so the fp64 mean sums in the same order), cached per column set."""
    bits = _bits(cohort, b)
    if cohort.n_models <= MAX_DEVICE_COLUMNS:
        return cohort.device(device), bits
    cols = tuple(int(i) for i in np.flatnonzero(bits))
    if len(cols) > MAX_DEVICE_COLUMNS:
        raise ValueError(f"an ensemble of {len(cols)} members exceeds the device sweep's "
                         f"{MAX_DEVICE_COLUMNS} columns")
    cache = cohort._dev.setdefault(("wide", device), {})
    dev = cache.get(cols)
    if dev is None:
        if len(cache) >= 16:
            cache.pop(next(iter(cache))).close()
        dev = cache[cols] = DeviceCohort(np.ascontiguousarray(cohort.scores[:, cols]), cohort.labels, device)
    return dev, np.ones(len(cols), np.uint8)


def ensemble_scores(cohort: Cohort, b: Selector, device: int = 0) -> np.ndarray:
    """Per-sample mean of the selected members' scores (device, column order fp64)."""
    dev, bits = _device_and_bits(cohort, b, device)
    return dev.ensemble(bits)[0]


def ensemble_roc_auc(cohort: Cohort, b: Selector, device: int = 0) -> float:
    """ROC-AUC of the ensemble mean: the accuracy profiler's value (device)."""
    dev, bits = _device_and_bits(cohort, b, device)
    return float(dev.auc_bits(bits[None, :])[0])


def accuracy_profile(cohort: Cohort, b: Selector, device: int = 0) -> AccuracyReport:
    """ROC-AUC / PR-AUC / F1 / accuracy of sigmoid(ensemble mean) at threshold 0.5."""
    from .metrics import f1_accuracy, pr_auc, roc_auc
    latent = ensemble_scores(cohort, b, device)
    prob = 1.0 / (1.0 + np.exp(-latent))
    f1, acc = f1_accuracy(cohort.labels, prob, threshold=0.5)
    return AccuracyReport(roc_auc=roc_auc(cohort.labels, prob, device), pr_auc=pr_auc(cohort.labels, prob),
                          f1=f1, accuracy=acc)


def record_cohort(zoo: ModelZoo, windows: np.ndarray, labels, *, selector: Selector | None = None, seed: int = 0,
                  batch: int = 1024, device: int = 0) -> Cohort:
    """Member logits over recorded windows -> Cohort (north star (4)).

    windows: [N, leads, W] raw samples (one recorded window per row, every
    lead); each member reads its own lead.  The windows run through the
    serving engine in tumbling mode (hop == W), `batch` rows per device tick.
    Columns follow zoo order; members outside `selector` (default: all) are
    not run and the cohort keeps only the selected columns.
    """
    from .engine import EnsembleEngine
    win = np.ascontiguousarray(windows, dtype=np.float32)
    if win.ndim != 3:
        raise ValueError("windows must be [N, leads, window]")
    N, leads, W = win.shape
    sel = selector if selector is not None else Selector.ones(zoo.n)
    P = max(1, min(batch, N))
    out = np.empty((N, sel.popcount))
    starts = list(range(0, N, P))

    def block(r0):
        chunk = win[r0:r0 + P]
        if chunk.shape[0] < P:
            chunk = np.concatenate([chunk, np.zeros((P - chunk.shape[0], leads, W), np.float32)])
        return np.ascontiguousarray(chunk)

    with EnsembleEngine(zoo, sel, P, leads=leads, fs=1, window_s=float(W), hop=W, seed=seed,
                        device=device) as eng:
        # pipelined: batch i+1 is submitted (copy + forward enqueued) before batch i is collected
        pending = [(starts[0], eng.submit(block(starts[0])))]
        for i in range(len(starts)):
            if i + 1 < len(starts):
                pending.append((starts[i + 1], eng.submit(block(starts[i + 1]))))
            r0, slot = pending.pop(0)
            res = eng.collect(slot)
            k = min(P, N - r0)
            out[r0:r0 + k] = res.member_logits[:k]
    return Cohort(labels=np.asarray(labels, np.int8), scores=out, seed=seed)


def save_cohort_csv(cohort: Cohort, path) -> None:
    """label,score_0..score_{n-1} rows, repr() floats (cohort.py:118-124)."""
    import csv
    with open(path, "w", newline="", encoding="utf-8") as fh:
        w = csv.writer(fh)
        w.writerow(["label"] + [f"score_{j}" for j in range(cohort.n_models)])
        w.writerows([int(lab)] + [repr(float(v)) for v in row] for lab, row in zip(cohort.labels, cohort.scores))
