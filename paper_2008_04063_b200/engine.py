"""`EnsembleEngine`: the per-tick predict call, backed by the C-ABI library.

One engine = one device context (`hb_ctx`) holding every (patient, lead)
stream's ring buffer, the selected members' fp16 weights and the per-tick CUDA
graph.  It replaces, for a whole tick of P patients at once:

* `Aggregator.add` buffering (`pkg/src/zooserve/runtime.py:98-115`) ->
  `ingest` / the append inside `tick`;
* `_WindowScorer.draw` (`runtime.py:131-136`) -> `tick`, which scores the real
  window of every patient with every selected member and returns per-member
  logits plus both aggregation conventions (mean of member sigmoids, and the
  reference's mean latent normalised by popcount, `cohort.py:89-97`);
* `service_time` (`latency.py:145-151`) -> the measured device time of a tick.

There is no CPU path: without the built library or a CUDA device every call
raises (`errors.DeviceError`).
"""

from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass
from functools import lru_cache

import numpy as np

from . import _lib, arch
from .errors import ConfigurationError, EmptyEnsembleError
from .zoo import ModelZoo, Selector, check_selector


@lru_cache(maxsize=256)
def _cached_params(width: int, depth: int, seed: int, member_id: str) -> np.ndarray:
    p = arch.member_params(width, depth, seed, member_id)
    return arch.flatten_params(p, width, depth)


def member_blob(profile, seed: int = 0) -> np.ndarray:
    """Flat fp32 parameter blob of a zoo member (deterministic per (seed, id))."""
    return _cached_params(profile.width, profile.depth, seed, profile.id)


@dataclass
class TickResult:
    member_ids: tuple          # selected member ids, zoo order
    member_logits: np.ndarray  # [P, M] float32
    ens_prob: np.ndarray       # [P] mean of member sigmoids (north star)
    ens_mean_logit: np.ndarray  # [P] mean latent / popcount (reference convention)


class EnsembleEngine:
    """Device-resident ensemble scorer for P patients x n_leads streams."""

    def __init__(self, zoo: ModelZoo, selector: Selector, patients: int, *, leads: int = 3, fs: int = 250,
                 window_s: float = 30.0, hop: int | None = None, seed: int = 0, device: int = 0,
                 keep_windows: bool = False, register: str = "selected"):
        check_selector(selector, zoo)
        if selector.popcount == 0:
            raise EmptyEnsembleError("cannot serve an empty ensemble")
        per_window = fs * window_s
        if abs(per_window - round(per_window)) > 1e-6 or round(per_window) < 1:
            raise ConfigurationError(f"rates: rate * window must be a positive integer, got {per_window}")
        self.zoo = zoo
        self.patients = int(patients)
        self.leads = int(leads)
        self.fs = int(fs)
        self.window = int(round(per_window))
        self.hop = int(hop) if hop is not None else self.window
        self.seed = seed
        self._lock = threading.Lock()
        L = _lib.lib()
        cfg = _lib.HbConfig(self.patients, self.leads, self.fs, self.window, self.hop, 0, int(keep_windows))
        h = C.c_void_p()
        _lib.check(L.hb_create(device, C.byref(cfg), C.byref(h)))
        self._h = h
        self._hb_tick = L.hb_tick
        self._hb_submit = L.hb_tick_submit
        self._hb_collect = L.hb_tick_collect
        self._next_slot = 0
        self._slot_ids: list = [None, None]  # member ids of the tick submitted into each slot
        self._out_ptrs = None  # (out, member_logits, ens_prob, ens_mean_logit addresses) of the last TickResult
        self._registered: set = set()
        to_register = range(zoo.n) if register == "all" else selector.indices()
        for i in to_register:
            self._register(i)
        self.selector = None
        self.set_selector(selector)

    # ------------------------------------------------------------------ setup
    def _register(self, i: int) -> None:
        prof = self.zoo.profiles[i]
        if prof.lead >= self.leads:
            raise ConfigurationError(f"rates: no stream configured for modality {prof.modality!r}")
        if prof.input_len != self.window:
            raise ConfigurationError(f"profile {prof.id!r}: input_len {prof.input_len} != window {self.window}")
        blob = member_blob(prof, self.seed)
        _lib.check(_lib.lib().hb_add_member(self._h, i, prof.lead, prof.width, prof.depth, _lib.fptr(blob),
                                            blob.size), self._h)
        self._registered.add(i)

    def set_selector(self, b: Selector) -> None:
        check_selector(b, self.zoo)
        if b.popcount == 0:
            raise EmptyEnsembleError("cannot serve an empty ensemble")
        with self._lock:
            for i in b.indices():
                if i not in self._registered:
                    self._register(i)
            bits = (C.c_uint8 * b.n)(*b.bits)
            _lib.check(_lib.lib().hb_set_selector(self._h, bits, b.n), self._h)
            self.selector = b
            self.member_ids = tuple(self.zoo.profiles[i].id for i in b.indices())
            self._out_ptrs = None

    # ------------------------------------------------------------------ data path
    def _check_block(self, samples, n) -> np.ndarray:
        a = np.ascontiguousarray(samples, dtype=np.float32)
        if a.shape != (self.patients, self.leads, n):
            raise ValueError(f"expected samples of shape {(self.patients, self.leads, n)}, got {a.shape}")
        return a

    def prepare(self) -> None:
        """Plan, capture and upload the tick graphs of the current selection now
        (`hb_prepare`), so the next tick is not charged the one-off setup."""
        with self._lock:
            _lib.check(_lib.lib().hb_prepare(self._h), self._h)

    def ingest(self, samples) -> None:
        """Append [P, leads, n] samples to every stream without scoring (warm-up / catch-up)."""
        a = np.ascontiguousarray(samples, dtype=np.float32)
        if a.ndim != 3 or a.shape[:2] != (self.patients, self.leads):
            raise ValueError(f"expected samples of shape ({self.patients}, {self.leads}, n), got {a.shape}")
        with self._lock:
            _lib.check(_lib.lib().hb_ingest(self._h, _lib.fptr(a), a.shape[2], None), self._h)

    def _ptrs_of(self, out: TickResult, M: int | None = None) -> tuple:
        M = self.selector.popcount if M is None else M
        for arr, shape in ((out.member_logits, (self.patients, M)),
                           (out.ens_prob, (self.patients,)), (out.ens_mean_logit, (self.patients,))):
            if arr.dtype != np.float32 or not arr.flags.c_contiguous or arr.shape != shape:
                raise ValueError(f"output buffers must be C-contiguous float32 of shape {shape}")
        return (out, out.member_logits.ctypes.data, out.ens_prob.ctypes.data, out.ens_mean_logit.ctypes.data)

    def tick(self, samples, out: TickResult | None = None) -> TickResult:
        """Append one hop [P, leads, hop] and score every patient's latest window.

        Per-call host overhead is kept to a few microseconds: a float32
        C-contiguous block of the right shape is passed as is, and the output
        buffers' addresses are cached per reused ``out`` (the serving loop and
        the benchmark reuse one TickResult)."""
        if (type(samples) is np.ndarray and samples.dtype == np.float32 and samples.flags.c_contiguous
                and samples.shape == (self.patients, self.leads, self.hop)):
            a = samples
        else:
            a = self._check_block(samples, self.hop)
        if out is None:
            M = self.selector.popcount
            out = TickResult(self.member_ids, np.empty((self.patients, M), np.float32),
                             np.empty(self.patients, np.float32), np.empty(self.patients, np.float32))
        cached = self._out_ptrs
        if cached is None or cached[0] is not out:
            cached = self._out_ptrs = self._ptrs_of(out)
        with self._lock:
            rc = self._hb_tick(self._h, a.ctypes.data, cached[1], cached[2], cached[3], None)
        if rc:
            _lib.check(rc, self._h)
        return out

    def submit(self, samples) -> int:
        """Pipelined tick, first half: enqueue the H2D of this hop, the tick and the D2H of its
        outputs into one of two pinned slots, and return the slot without waiting.  Submit tick
        t+1 before ``collect``-ing tick t and the device never idles on the host round trip.
        Ticks run in submission order (one stream per engine)."""
        if (type(samples) is np.ndarray and samples.dtype == np.float32 and samples.flags.c_contiguous
                and samples.shape == (self.patients, self.leads, self.hop)):
            a = samples
        else:
            a = self._check_block(samples, self.hop)
        slot = self._next_slot
        with self._lock:
            rc = self._hb_submit(self._h, a.ctypes.data, slot, None)
            if rc:
                _lib.check(rc, self._h)
            self._slot_ids[slot] = self.member_ids
        self._next_slot = slot ^ 1
        return slot

    def collect(self, slot: int, out: TickResult | None = None) -> TickResult:
        """Pipelined tick, second half: wait for the tick submitted into ``slot`` and return its outputs
        (labelled with the members that tick was submitted with)."""
        ids = self._slot_ids[slot] if slot in (0, 1) and self._slot_ids[slot] is not None else self.member_ids
        if out is None:
            out = TickResult(ids, np.empty((self.patients, len(ids)), np.float32),
                             np.empty(self.patients, np.float32), np.empty(self.patients, np.float32))
        cached = self._out_ptrs
        if cached is None or cached[0] is not out:
            cached = self._out_ptrs = self._ptrs_of(out, len(ids))
        with self._lock:
            rc = self._hb_collect(self._h, slot, cached[1], cached[2], cached[3])
            if rc:
                _lib.check(rc, self._h)
            self._slot_ids[slot] = None
        return out

    def stage_device(self, dev_ptr: int, stream: int | None = None) -> None:
        _lib.check(_lib.lib().hb_stage_device(self._h, C.c_void_p(dev_ptr), C.c_void_p(stream or 0) if stream else None),
                   self._h)

    def tick_device(self, stream: int | None = None) -> None:
        """Tick with inputs already staged on the device; outputs stay on the device."""
        _lib.check(_lib.lib().hb_tick_device(self._h, C.c_void_p(stream) if stream else None), self._h)

    def device_outputs(self) -> tuple[int, int, int]:
        ml, ep, el = C.c_void_p(), C.c_void_p(), C.c_void_p()
        _lib.check(_lib.lib().hb_device_outputs(self._h, C.byref(ml), C.byref(ep), C.byref(el)), self._h)
        return ml.value, ep.value, el.value

    def last_windows(self) -> tuple[np.ndarray, np.ndarray]:
        """Raw windows [P, leads, W] and (mean, std) [P, leads, 2] of the latest tick (keep_windows=True)."""
        raw = np.empty((self.patients, self.leads, self.window), np.float32)
        stats = np.empty((self.patients, self.leads, 2), np.float32)
        _lib.check(_lib.lib().hb_last_windows(self._h, _lib.fptr(raw), _lib.fptr(stats), None), self._h)
        return raw, stats

    def last_normalized(self) -> np.ndarray:
        """The z-normalised fp16 windows [leads, P, W] the latest tick's members consumed."""
        out = np.empty((self.leads, self.patients, self.window), np.float16)
        _lib.check(_lib.lib().hb_last_normalized(self._h, C.c_void_p(out.ctypes.data), None), self._h)
        return out

    def profile_tick(self, stream: int | None = None, cap: int = 4096):
        """Per-launch (kind, ms, flops, bytes) of one eagerly launched tick (advances the stream)."""
        kinds = np.zeros(cap, np.int32)
        ms = np.zeros(cap, np.float32)
        fl = np.zeros(cap, np.float64)
        by = np.zeros(cap, np.float64)
        n = _lib.lib().hb_profile_tick(self._h, C.c_void_p(stream) if stream else None, cap,
                                       kinds.ctypes.data_as(C.POINTER(C.c_int)), _lib.fptr(ms),
                                       fl.ctypes.data_as(C.POINTER(C.c_double)),
                                       by.ctypes.data_as(C.POINTER(C.c_double)))
        if n < 0:
            _lib.check(-n, self._h)
        n = min(n, cap)
        return kinds[:n], ms[:n], fl[:n], by[:n]

    def last_tick_seconds(self) -> float:
        """Device seconds of the most recent tick graph (CUDA events on its stream)."""
        ms = C.c_float()
        _lib.check(_lib.lib().hb_last_tick_ms(self._h, C.byref(ms)), self._h)
        return ms.value / 1e3

    def time_tick(self, reps: int = 5) -> float:
        """Median device seconds of `reps` tick launches (measurement only; advances the stream)."""
        ms = C.c_float()
        with self._lock:
            _lib.check(_lib.lib().hb_time_tick(self._h, int(reps), C.byref(ms)), self._h)
        return ms.value / 1e3

    def tick_work(self) -> tuple[float, float]:
        """(conv FLOPs, activation bytes) of one tick for the current selector."""
        f, b = C.c_double(), C.c_double()
        _lib.check(_lib.lib().hb_tick_work(self._h, C.byref(f), C.byref(b)), self._h)
        return f.value, b.value

    def close(self) -> None:
        if getattr(self, "_h", None):
            _lib.lib().hb_destroy(self._h)
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
