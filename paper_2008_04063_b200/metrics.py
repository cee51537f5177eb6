"""Classification metrics of the drop-in surface.

`roc_auc` / `roc_auc_many` keep the reference's signatures, validation and
exceptions (`pkg/src/zooserve/metrics.py:16-76`) but are computed by the K6
sweep kernel (`csrc/sweep.cu`): exact Mann-Whitney U from midranks with half
credit for ties, so values are bit-identical to the reference's.  There is no
CPU fallback for them.

`pr_auc` and `f1_accuracy` (`metrics.py:79-111`) only feed the one-off
accuracy report (`cohort.accuracy_profile`), never a per-tick or
per-candidate path, so they stay plain numpy on the host.
"""

from __future__ import annotations

import numpy as np

from .errors import UndefinedMetricError


def validate(labels, scores) -> tuple[np.ndarray, np.ndarray]:
    """1-D, same length, non-empty, labels in {0,1}, finite scores (metrics.py:16-27)."""
    lab = np.asarray(labels)
    sc = np.asarray(scores, dtype=np.float64)
    if lab.ndim != 1 or lab.shape != sc.shape:
        raise ValueError("labels and scores must be 1-D and the same length")
    if lab.size == 0:
        raise ValueError("need at least one sample")
    if not np.isin(lab, (0, 1)).all():
        raise ValueError("labels must be 0 or 1")
    if not np.isfinite(sc).all():
        raise ValueError("scores must be finite")
    return lab.astype(np.int8), sc


def _both_classes(lab: np.ndarray) -> None:
    pos = int(lab.sum())
    if pos == 0 or pos == lab.size:
        raise UndefinedMetricError("roc_auc needs both classes present")


def roc_auc(labels, scores, device: int = 0) -> float:
    """P(score_pos > score_neg) + 0.5 P(tie), on the device."""
    from .cohort import DeviceCohort
    lab, sc = validate(labels, scores)
    _both_classes(lab)
    with DeviceCohort(sc[:, None], lab, device=device) as dc:
        return float(dc.auc_bits(np.ones((1, 1), np.uint8))[0])


def roc_auc_many(labels, score_matrix, device: int = 0) -> np.ndarray:
    """roc_auc of every column against shared labels (metrics.py:63-76), one device pass."""
    from .cohort import DeviceCohort
    lab = np.asarray(labels).astype(np.int8)
    mat = np.asarray(score_matrix, dtype=np.float64)
    if mat.ndim != 2 or mat.shape[0] != lab.size:
        raise ValueError("score_matrix must be (n_samples, n_columns)")
    _both_classes(lab)
    out = np.empty(mat.shape[1])
    step = 256
    for c0 in range(0, mat.shape[1], step):
        block = np.ascontiguousarray(mat[:, c0:c0 + step])
        k = block.shape[1]
        with DeviceCohort(block, lab, device=device) as dc:
            out[c0:c0 + k] = dc.auc_bits(np.eye(k, dtype=np.uint8))
    return out


def pr_auc(labels, scores) -> float:
    """Average precision: step curve over descending score, tied scores enter together."""
    lab, sc = validate(labels, scores)
    n_pos = int(lab.sum())
    if n_pos == 0:
        raise UndefinedMetricError("pr_auc needs at least one positive")
    order = np.argsort(-sc, kind="stable")
    y, s = lab[order].astype(np.float64), sc[order]
    tp, fp = np.cumsum(y), np.cumsum(1.0 - y)
    keep = np.r_[s[1:] != s[:-1], True]     # last sample of every distinct score
    tp, fp = tp[keep], fp[keep]
    recall = tp / n_pos
    return float(np.dot(np.diff(recall, prepend=0.0), tp / (tp + fp)))


def f1_accuracy(labels, scores, threshold: float = 0.5) -> tuple[float, float]:
    """(F1, accuracy) of the predictions score > threshold; F1 is 0 when undefined."""
    lab, sc = validate(labels, scores)
    pred, actual = sc > threshold, lab == 1
    tp = int(np.sum(pred & actual))
    wrong = int(np.sum(pred != actual))
    denom = 2 * tp + wrong
    return ((2 * tp / denom) if denom else 0.0), float(np.mean(pred == actual))


def r2(predicted, actual) -> float:
    """Coefficient of determination 1 - SS_res / SS_tot (metrics.py:114-127): 1-D, equal length,
    >= 2 samples; constant actuals raise UndefinedMetricError."""
    pr = np.asarray(predicted, dtype=np.float64)
    ac = np.asarray(actual, dtype=np.float64)
    if pr.ndim != 1 or pr.shape != ac.shape:
        raise ValueError("predicted and actual must be 1-D and the same length")
    if ac.size < 2:
        raise ValueError("need at least two samples")
    centred = ac - ac.mean()
    ss_tot = float(np.sum(centred * centred))
    if ss_tot == 0.0:
        raise UndefinedMetricError("r2 undefined for constant actuals")
    resid = ac - pr
    return 1.0 - float(np.sum(resid * resid)) / ss_tot


def sweep_auc(labels, score_matrix, selectors, device: int = 0) -> np.ndarray:
    """AUC of the ensemble mean of every selector, one shot through the C-ABI's `hb_sweep_auc`
    (the batched accuracy pass of `exhaustive_search`, composer.py:614-619): `selectors` are
    ints whose bit k selects column k (LSB = model 0, composer.py:616), n <= 32 columns."""
    import ctypes as C

    from . import _lib
    lab, _ = validate(labels, np.zeros(len(labels)))
    mat = np.ascontiguousarray(score_matrix, dtype=np.float64)
    if mat.ndim != 2 or mat.shape[0] != lab.size:
        raise ValueError("score_matrix must be (n_samples, n_columns)")
    sel = np.ascontiguousarray(selectors, dtype=np.uint32)
    out = np.empty(sel.size, np.float64)
    rc = _lib.lib().hb_sweep_auc(device, _lib.dptr(mat), lab.ctypes.data_as(C.POINTER(C.c_int8)), mat.shape[0],
                                 mat.shape[1], sel.ctypes.data_as(C.POINTER(C.c_uint32)), sel.size, _lib.dptr(out))
    _lib.check(rc, None, "hb_cohort_last_error")
    return out
