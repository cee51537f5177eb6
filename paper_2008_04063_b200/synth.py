"""Seeded synthetic 250 Hz ECG streams (there is no dataset).

Each (patient, lead) stream is a deterministic float32 function of the absolute
sample index: Gaussian QRS-like pulses at a per-patient heart rate in
[1.0, 2.6] Hz with per-patient QRS width / T-wave shape, a 0.3 Hz baseline
wander and Gaussian noise of per-patient level.  Noise is drawn
per 1-second chunk from `derive_seed(seed, "ecg", patient, lead, chunk)`, so
any chunk-aligned slice of a stream is reproducible on its own — the ingest
path, the CPU oracle and the reference `Aggregator` all see identical samples.

`zero_stream` is the reference's own wall-clock generator signal (every value
0.0, `pkg/src/zooserve/runtime.py:358`); it exercises the z-norm zero-variance
guard.
"""

from __future__ import annotations

import numpy as np

from .seeds import derive_seed

FS = 250
CHUNK = FS  # noise chunk = 1 s


def _patient_params(seed: int, patient: int) -> dict:
    r = np.random.default_rng(derive_seed(seed, "ecg-patient", patient))
    return {
        "hr": r.uniform(1.0, 2.6),            # beats/s (60-156 bpm)
        "phase": r.uniform(0.0, 1.0),
        "qrs": r.uniform(0.008, 0.025),       # QRS gaussian width, s
        "t_amp": r.uniform(0.05, 0.5),        # T-wave amplitude (relative)
        "t_delay": r.uniform(0.15, 0.3),
        "wander": r.uniform(0.02, 0.4),       # 0.3 Hz baseline wander amplitude
        "wphase": r.uniform(0.0, 2 * np.pi),
        "noise": r.uniform(0.02, 0.12),
    }


def ecg_samples(seed: int, patient: int, lead: int, start: int, count: int,
                fs: int = FS) -> np.ndarray:
    """Samples [start, start+count) of stream (patient, lead) as float32."""
    if count <= 0:
        return np.zeros(0, np.float32)
    pp = _patient_params(seed, patient)
    amp = (1.0, 1.4, 0.8)[lead % 3]
    t = np.arange(start, start + count, dtype=np.float64) / fs
    period = 1.0 / pp["hr"]
    phase = pp["phase"] * period
    k = np.round((t - phase) / period)
    dt = t - (phase + k * period)              # distance to the nearest beat centre
    sig = amp * np.exp(-0.5 * (dt / pp["qrs"]) ** 2)
    sig += amp * pp["t_amp"] * np.exp(-0.5 * ((dt - pp["t_delay"]) / 0.04) ** 2)
    sig += pp["wander"] * np.sin(2 * np.pi * 0.3 * t + pp["wphase"] + lead)
    c0, c1 = start // CHUNK, (start + count - 1) // CHUNK
    noise = np.concatenate([
        np.random.default_rng(derive_seed(seed, "ecg", patient, lead, c)).standard_normal(CHUNK)
        for c in range(c0, c1 + 1)])
    off = start - c0 * CHUNK
    sig += pp["noise"] * noise[off:off + count]
    return sig.astype(np.float32)


def ecg_block(seed: int, patients, leads: int, start: int, count: int) -> np.ndarray:
    """[P, leads, count] float32 block of all streams (a tick's ingest payload)."""
    patients = list(range(patients)) if isinstance(patients, int) else list(patients)
    out = np.empty((len(patients), leads, count), np.float32)
    for i, p in enumerate(patients):
        for l in range(leads):
            out[i, l] = ecg_samples(seed, p, l, start, count)
    return out


def zero_stream(count: int) -> np.ndarray:
    return np.zeros(count, np.float32)
