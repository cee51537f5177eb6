"""ORACLE (test infrastructure only) — CPU restatement of stream windowing.

Restates the reference's per-(patient, modality) `Aggregator`
(`pkg/src/zooserve/runtime.py:76-115`): samples accumulate until exactly
rate*window of them arrived, then window k = samples [k*W, (k+1)*W) is emitted
with `window_start_s = k * window_s` and `t_flush` = the last sample's time;
`rate*window` must be a positive integer (`runtime.py:85-89`).  The sliding
generalisation used by the B200 ring buffer (hop h < W) is the window ending at
every multiple of h; at h == W it reduces to the tumbling Aggregator exactly —
`tests/test_golden.py` pins both against windows the reference produced.
"""

from __future__ import annotations

import numpy as np


def samples_per_window(rate_qps: float, window_s: float) -> int:
    per = rate_qps * window_s
    if abs(per - round(per)) > 1e-6 or round(per) < 1:
        raise ValueError(f"rate * window must be a positive integer, got {per}")
    return int(round(per))


def tumbling_windows(stream: np.ndarray, W: int):
    """Reference Aggregator semantics: [(k, samples[kW:(k+1)W]) for every complete window]."""
    n = len(stream) // W
    return [(k, np.asarray(stream[k * W:(k + 1) * W])) for k in range(n)]


def sliding_window(stream: np.ndarray, end: int, W: int) -> np.ndarray:
    """The window the device ring holds after `end` samples: stream[end-W:end] (zeros before 0)."""
    out = np.zeros(W, dtype=np.asarray(stream).dtype)
    lo = end - W
    src = np.asarray(stream[max(lo, 0):end])
    out[W - len(src):] = src
    return out


def window_times(k: int, window_s: float, rate_qps: float, W: int) -> tuple[float, float]:
    """(window_start_s, t_flush) of window k when sample i is generated at t = (i+1)/rate
    (the reference's wall-clock schedule, `runtime.py:349-353`)."""
    return k * window_s, ((k + 1) * W) / rate_qps
