"""Ensemble selection over GPU-backed profilers.

Drop-in pieces of `pkg/src/zooserve/composer.py`:
  ProfileRecord / SearchParams / SearchResult      composer.py:44-143
  constraint_penalty, objective_value, dual_...    composer.py:146-167
  Profilers, make_accuracy_profiler                composer.py:270-302
  exhaustive_search                                composer.py:597-638

`exhaustive_search` scores every non-empty selector's accuracy in ONE device
pass (K6, `hb_cohort_auc_range`) instead of the reference's fp64 BLAS matmul +
per-column argsort, then walks the candidates in enumeration order with the
reference's objective and tie-break (strict improvement keeps the first,
i.e. lowest selector value).  Selection and AUCs are bit-identical to the
reference (tests/golden/sweep_*.npz).

The SMBO loop, genetic exploration and the RD/AF/LF/NPO baselines are a
sequential, tiny-data CPU search (out of scope); they consume
these profilers unchanged through the `Profilers` callables — pass
`make_accuracy_profiler(cohort)` and any latency callable to the reference's
`smbo_search`.
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass
from typing import Callable

import numpy as np

from .cohort import Cohort, ensemble_roc_auc
from .latency import SystemConfig
from .zoo import ModelZoo, Selector

HARD = "hard"
SOFT = "soft"
LATENCY_SURROGATE_CAP_S = 1e3


@dataclass(frozen=True)
class ProfileRecord:
    b: Selector
    accuracy: float
    latency_s: float

    def __post_init__(self):
        if not 0.0 <= self.accuracy <= 1.0:
            raise ValueError("accuracy must lie in [0, 1]")
        if self.latency_s < 0:
            raise ValueError("latency must be non-negative")


@dataclass(frozen=True)
class SearchParams:
    latency_weight: float = 1.0
    n_iters: int = 20
    n_warm: int = 20
    n_explore: int = 200
    top_k: int = 5
    mutation_degree: int = 2
    p_genetic: float = 0.8
    p_mutation: float = 0.5
    constraint_mode: str = HARD
    seed: int = 0

    def __post_init__(self):
        if self.latency_weight < 0:
            raise ValueError("latency_weight must be >= 0")
        if self.n_iters < 0 or min(self.n_warm, self.n_explore, self.top_k) < 1:
            raise ValueError("n_iters >= 0 and n_warm/n_explore/top_k >= 1 required")
        if self.top_k > self.n_explore:
            raise ValueError("top_k must not exceed n_explore")
        if not (0 <= self.p_genetic <= 1 and 0 <= self.p_mutation <= 1):
            raise ValueError("probabilities must lie in [0, 1]")
        if self.mutation_degree < 0:
            raise ValueError("mutation_degree must be >= 0")
        if self.constraint_mode not in (HARD, SOFT):
            raise ValueError(f"constraint_mode must be '{HARD}' or '{SOFT}'")


@dataclass(frozen=True)
class TrajectoryPoint:
    iteration: int
    best_accuracy: float
    best_latency_s: float
    best_objective: float


def _finite_or_none(x: float):
    return x if math.isfinite(x) else None


@dataclass
class SearchResult:
    best: Selector
    best_objective: float
    best_accuracy: float
    best_latency_s: float
    trajectory: list
    profiled: list
    profiler_calls: int

    @property
    def feasible(self) -> bool:
        return math.isfinite(self.best_objective)

    def to_json_dict(self) -> dict:
        return {
            "best": str(self.best),
            "best_objective": _finite_or_none(self.best_objective),
            "best_accuracy": self.best_accuracy,
            "best_latency_s": _finite_or_none(self.best_latency_s),
            "feasible": self.feasible,
            "profiler_calls": self.profiler_calls,
            "trajectory": [{"iteration": p.iteration, "best_accuracy": p.best_accuracy,
                            "best_latency_s": _finite_or_none(p.best_latency_s),
                            "best_objective": _finite_or_none(p.best_objective)} for p in self.trajectory],
            "profiled": [{"b": str(r.b), "accuracy": r.accuracy, "latency_s": _finite_or_none(r.latency_s)}
                         for r in self.profiled],
        }

    def save_json(self, path) -> None:
        with open(path, "w", encoding="utf-8") as fh:
            json.dump(self.to_json_dict(), fh, indent=2, sort_keys=True)
            fh.write("\n")

    def save_trajectory_csv(self, path) -> None:
        """iter,best_acc,best_lat,best_obj rows with repr() floats (composer.py:138-143)."""
        rows = ["iter,best_acc,best_lat,best_obj"]
        rows += [f"{p.iteration},{p.best_accuracy!r},{p.best_latency_s!r},{p.best_objective!r}"
                 for p in self.trajectory]
        with open(path, "w", encoding="utf-8") as fh:
            fh.write("\n".join(rows) + "\n")


def constraint_penalty(x: float, mode: str = HARD, weight: float = 1.0) -> float:
    """Penalty of constraint slack x: -inf below zero (hard) or weight * x (soft).  The hard test is
    `x < 0` as in the reference (composer.py:146-152): a NaN slack (inf budget - inf latency) is 0."""
    if mode == HARD:
        return -math.inf if x < 0 else 0.0
    if mode == SOFT:
        return weight * x
    raise ValueError(f"unknown constraint mode {mode!r}")


def objective_value(rec: ProfileRecord, budget_s: float, params: SearchParams) -> float:
    return rec.accuracy + constraint_penalty(budget_s - rec.latency_s, params.constraint_mode,
                                             params.latency_weight)


def dual_objective_value(rec: ProfileRecord, accuracy_floor: float, params: SearchParams) -> float:
    return rec.latency_s - constraint_penalty(rec.accuracy - accuracy_floor, params.constraint_mode,
                                              params.latency_weight)


class Profilers:
    """Memoising pair of true profilers; `calls` = distinct selectors profiled."""

    def __init__(self, accuracy_fn: Callable[[Selector], float], latency_fn: Callable[[Selector], float]):
        self._acc, self._lat = accuracy_fn, latency_fn
        self._cache: dict = {}

    @property
    def calls(self) -> int:
        return len(self._cache)

    def known(self, b: Selector) -> bool:
        return b in self._cache

    def profile(self, b: Selector) -> ProfileRecord:
        if b not in self._cache:
            self._cache[b] = ProfileRecord(b=b, accuracy=self._acc(b), latency_s=self._lat(b))
        return self._cache[b]

    def records(self) -> list:
        return list(self._cache.values())


def make_accuracy_profiler(cohort: Cohort, device: int = 0) -> Callable[[Selector], float]:
    """f_a(b) = device ROC-AUC of the ensemble mean over the cohort."""
    return lambda b: ensemble_roc_auc(cohort, b, device)


def sweep_aucs(cohort: Cohort, device: int = 0, chunk: int = 1 << 22) -> np.ndarray:
    """AUC of every non-empty selector, enumeration order (values 1 .. 2^n - 1)."""
    n = cohort.n_models
    if n > 30:
        raise ValueError("enumerating every selector needs n <= 30")
    total = (1 << n) - 1
    dev = cohort.device(device)
    out = np.empty(total)
    for v0 in range(1, total + 1, chunk):
        cnt = min(chunk, total - v0 + 1)
        out[v0 - 1:v0 - 1 + cnt] = dev.auc_range(v0, cnt)
    return out


def exhaustive_search(zoo: ModelZoo, cohort: Cohort, latency_profiler, budget_s: float,
                      sys: SystemConfig | None = None, params: SearchParams | None = None,
                      accuracy_floor: float | None = None, device: int = 0) -> SearchResult:
    """Every non-empty selector with the true profilers (n <= 20), accuracies from one device sweep.

    With `accuracy_floor` the dual problem (minimise latency) is solved.  Ties
    keep the lowest selector value (enumeration order, composer.py:624-631).
    """
    if zoo.n > 20:
        raise ValueError(f"exhaustive search is guarded to n <= 20, got {zoo.n}")
    if zoo.n == 0:
        raise ValueError("zoo must be non-empty")
    params = params if params is not None else SearchParams()
    if cohort.n_models != zoo.n:
        raise ValueError(f"selector length {zoo.n} does not match cohort width {cohort.n_models}")
    aucs = sweep_aucs(cohort, device)
    n = zoo.n
    minimize = accuracy_floor is not None
    records = []
    best_rec, best_val = None, None
    for v in range(1, 1 << n):
        b = Selector.from_int(n, v)
        rec = ProfileRecord(b=b, accuracy=float(aucs[v - 1]), latency_s=latency_profiler(b))
        records.append(rec)
        val = dual_objective_value(rec, accuracy_floor, params) if minimize else objective_value(rec, budget_s,
                                                                                                 params)
        if best_rec is None or (val < best_val if minimize else val > best_val):
            best_rec, best_val = rec, val
    traj = [TrajectoryPoint(0, best_rec.accuracy, best_rec.latency_s, best_val)]
    return SearchResult(best=best_rec.b, best_objective=best_val, best_accuracy=best_rec.accuracy,
                        best_latency_s=best_rec.latency_s, trajectory=traj, profiled=records,
                        profiler_calls=len(records))
