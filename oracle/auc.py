"""ORACLE (test infrastructure only) — CPU restatement of the profiler sweep.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU legs may import
this module, as the checker / CPU baseline; the product path never does.

Parity: PINNED.  `tests/test_oracle_golden.py` checks every function here
against outputs of the reference itself (tests/golden/*, made by
tools/make_golden.py from /root/reference/pkg/src/zooserve).

Restated algorithms:
  * midrank rank-sum AUC, ties averaged      (metrics.py:30-60)
    AUC = (R_pos - n_pos(n_pos+1)/2) / (n_pos n_neg)
  * roc_auc_many over columns                 (metrics.py:63-76)
  * exhaustive sweep: ens = scores @ bits.T / popcount, candidate values
    1 .. 2^n-1 with bit k <-> column k (LSB = column 0)   (composer.py:614-619)
    — restated as a column-ordered fp64 sum (what the K6 kernel computes; see
    csrc/sweep.cu for why this reproduces the reference's AUCs exactly).
"""

from __future__ import annotations

import numpy as np


def pos_rank_sum(labels: np.ndarray, scores: np.ndarray) -> float:
    """Sum of the positives' 1-based midranks (tied scores share the mean rank)."""
    labels = np.asarray(labels, np.int64)
    scores = np.asarray(scores, np.float64)
    order = np.argsort(scores, kind="stable")
    s = scores[order]
    lab = labels[order]
    n = s.size
    # run boundaries of equal scores
    starts = np.flatnonzero(np.r_[True, s[1:] != s[:-1]])
    ends = np.r_[starts[1:], n]                      # exclusive
    mid = (starts + ends + 1) / 2.0                  # mean of 1-based ranks start+1 .. end
    run_of = np.repeat(np.arange(starts.size), ends - starts)
    return float(np.dot(lab, mid[run_of]))


def roc_auc(labels, scores) -> float:
    labels = np.asarray(labels, np.int64)
    n_pos = int(labels.sum())
    n_neg = labels.size - n_pos
    if n_pos == 0 or n_neg == 0:
        raise ValueError("roc_auc needs both classes present")
    u = pos_rank_sum(labels, scores) - n_pos * (n_pos + 1) / 2.0
    return u / (n_pos * n_neg)


def roc_auc_many(labels, matrix) -> np.ndarray:
    m = np.asarray(matrix, np.float64)
    return np.array([roc_auc(labels, m[:, j]) for j in range(m.shape[1])])


def ensemble_mean(scores: np.ndarray, cols) -> np.ndarray:
    """Column-ordered fp64 sum of the selected columns divided by their count."""
    acc = np.zeros(scores.shape[0])
    for k in cols:
        acc = acc + scores[:, k]
    return acc / float(len(cols))


def sweep(labels, scores, values) -> np.ndarray:
    """AUC of every candidate (integer selector values, bit k <-> column k)."""
    scores = np.asarray(scores, np.float64)
    n = scores.shape[1]
    out = np.empty(len(values))
    for i, v in enumerate(values):
        cols = [k for k in range(n) if (int(v) >> k) & 1]
        out[i] = roc_auc(labels, ensemble_mean(scores, cols))
    return out
