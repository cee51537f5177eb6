"""ORACLE (test infrastructure + CPU baseline only) — one serving tick on the CPU.

The whole hot path restated on the host: gather each patient's latest window
(`windows.sliding_window`, = the reference `Aggregator` at hop == window,
`pkg/src/zooserve/runtime.py:98-115`), z-normalise, run every selected member
(`cnn.member_forward`, PyTorch fp32 on all host threads) and aggregate in zoo
order (mean latent / popcount as `cohort.py:89-97`, plus mean of sigmoids).
`bench.py` times this as the CPU baseline ("port" — the reference has no CNN to
run); the GPU parity tests use it as the checker.

Parameters: the oracle consumes the same flat fp32 blob the product hands to
`hb_add_member` (synthesised by `arch.member_params`, an INPUT generator like
`synth.ecg_block`), decoded with the oracle's own layer table (`cnn.unflatten`).
"""

from __future__ import annotations

import numpy as np

from paper_2008_04063_b200 import arch

from . import cnn, windows

_PARAMS: dict = {}


def member_blob(profile, seed: int = 0) -> np.ndarray:
    """The flat parameter blob of a zoo member (what `hb_add_member` receives)."""
    p = arch.member_params(profile.width, profile.depth, seed, profile.id)
    return arch.flatten_params(p, profile.width, profile.depth)


def params_for(profile, seed: int = 0, window: int = 7500) -> dict:
    key = (profile.width, profile.depth, seed, profile.id, window)
    if key not in _PARAMS:
        _PARAMS[key] = cnn.unflatten(member_blob(profile, seed), profile.width, profile.depth, window)
    return _PARAMS[key]


def member_windows(streams: np.ndarray, lead: int, end: int, window: int = 7500, beds=None) -> np.ndarray:
    beds = range(streams.shape[0]) if beds is None else beds
    return np.stack([windows.sliding_window(streams[p, lead], end, window) for p in beds])


def cpu_tick(zoo, selector, streams: np.ndarray, end: int, window: int = 7500, seed: int = 0, beds=None):
    """streams [P, leads, n] -> (member_logits [B, M], ens_prob [B], ens_mean_logit [B]) for the
    beds `beds` (default: all P)."""
    logits = []
    for i in selector.indices():
        prof = zoo.profiles[i]
        win = member_windows(streams, prof.lead, end, window, beds)
        logits.append(cnn.member_forward(cnn.znorm(win), params_for(prof, seed, window), prof.width, prof.depth))
    ml = np.stack(logits, axis=1)
    prob, mean_logit = cnn.ensemble(ml)
    return ml, prob, mean_logit
