"""ORACLE (test infrastructure + CPU baseline only) — one serving tick on the CPU.

The whole hot path restated on the host: gather each patient's latest window
(`windows.sliding_window`, = the reference `Aggregator` at hop == window,
`pkg/src/zooserve/runtime.py:98-115`), z-normalise, run every selected member
(`cnn.member_forward`, PyTorch fp32 on all host threads) and aggregate in zoo
order (mean latent / popcount as `cohort.py:89-97`, plus mean of sigmoids).
`bench.py` times this as the CPU baseline ("port" — the reference has no CNN to
run); the GPU parity tests use it as the checker.
"""

from __future__ import annotations

import numpy as np

from paper_2008_04063_b200 import arch

from . import cnn, windows

_PARAMS: dict = {}


def params_for(profile, seed: int = 0) -> dict:
    key = (profile.width, profile.depth, seed, profile.id)
    if key not in _PARAMS:
        _PARAMS[key] = arch.member_params(profile.width, profile.depth, seed, profile.id)
    return _PARAMS[key]


def cpu_tick(zoo, selector, streams: np.ndarray, end: int, window: int = 7500, seed: int = 0):
    """streams [P, leads, n] -> (member_logits [P, M], ens_prob [P], ens_mean_logit [P])."""
    P = streams.shape[0]
    logits = []
    for i in selector.indices():
        prof = zoo.profiles[i]
        win = np.stack([windows.sliding_window(streams[p, prof.lead], end, window) for p in range(P)])
        logits.append(cnn.member_forward(cnn.znorm(win), params_for(prof, seed), prof.width, prof.depth))
    ml = np.stack(logits, axis=1)
    prob, mean_logit = cnn.ensemble(ml)
    return ml, prob, mean_logit
