"""Serving path: windows, queries, the tick loop and its traces.

Drop-in for the serving half of `pkg/src/zooserve/runtime.py`:

  SensorSample / WindowBatch / QueryTrace        runtime.py:39-73
  Aggregator (host, per-sample)                  runtime.py:76-115
  run_simulation                                 runtime.py:153-235
  e2e_percentiles                                runtime.py:238-251

`run_simulation` keeps the reference's signature and, by default, its
deterministic discrete-event semantics — including the binormal score
stand-in `_WindowScorer` (runtime.py:118-136) and the analytic service time —
so existing callers get bit-identical traces (tests/golden/traces.json).
Passing `scorer=EngineScorer(...)` swaps that stand-in for the real thing:
every window boundary is ONE device tick (ring append -> window gather +
z-norm -> every selected member's ResNet forward -> aggregate, captured as a
CUDA graph, `engine.py`) over all patients' actual samples, the traces carry
the real member logits, and the service time is the measured device time of
that tick.  With `hop < window` the engine scores a sliding window every hop.
"""

from __future__ import annotations

import heapq
import json
import math
from collections import deque
from dataclasses import asdict, dataclass

import numpy as np

from .errors import ConfigurationError, EmptyEnsembleError
from .latency import ExecutorModel, service_time
from .zoo import ModelZoo, Selector, check_selector, modality_lead

DEFAULT_AGG_OVERHEAD_S = 0.002


@dataclass(frozen=True)
class SensorSample:
    patient_id: int
    modality: str
    t_gen: float
    value: float


@dataclass
class WindowBatch:
    patient_id: int
    modality: str
    window_start_s: float
    samples: np.ndarray
    t_flush: float

    def __post_init__(self):
        self.samples = np.asarray(self.samples, dtype=np.float64)


@dataclass(frozen=True)
class QueryTrace:
    query_id: int
    patient_id: int
    t_ingest: float
    t_enqueue: float
    t_dequeue: float
    t_done: float
    model_scores: dict
    ensemble_score: float

    def __post_init__(self):
        if not self.t_ingest <= self.t_enqueue <= self.t_dequeue <= self.t_done:
            raise ValueError("trace timestamps must be ordered ingest <= enqueue <= dequeue <= done")


def samples_per_window(modality: str, rate_qps: float, window_s: float) -> int:
    per = rate_qps * window_s
    if abs(per - round(per)) > 1e-6 or round(per) < 1:
        raise ConfigurationError(f"rates.{modality}: rate * window must be a positive integer, got {per}")
    return int(round(per))


class Aggregator:
    """Host-side tumbling buffer of one (patient, modality) stream.

    Emits window k = samples [kW, (k+1)W) once its last sample arrives
    (`window_start_s = k * window_s`, `t_flush` = that sample's time).  The
    device path does the same for every stream at once in its ring buffers
    (`EnsembleEngine.ingest` / `tick`); this class serves per-sample callers.
    """

    def __init__(self, patient_id: int, modality: str, rate_qps: float, window_s: float):
        self.patient_id, self.modality, self.window_s = patient_id, modality, window_s
        self.samples_per_window = samples_per_window(modality, rate_qps, window_s)
        self._buf = np.empty(self.samples_per_window)
        self._fill = 0
        self._k = 0
        self._last_t = -math.inf

    def add(self, sample: SensorSample):
        if sample.t_gen < self._last_t:
            raise ValueError(f"samples for ({self.patient_id}, {self.modality}) must arrive in time order")
        self._last_t = sample.t_gen
        self._buf[self._fill] = sample.value
        self._fill += 1
        if self._fill < self.samples_per_window:
            return None
        out = WindowBatch(self.patient_id, self.modality, self._k * self.window_s, self._buf.copy(), sample.t_gen)
        self._fill = 0
        self._k += 1
        return out


def _positive_shift(auc: float) -> float:
    from .cohort import positive_shift
    return positive_shift(auc)


class BinormalScorer:
    """The reference's inference stand-in (`_WindowScorer`, runtime.py:118-136),
    kept so `run_simulation` without a device scorer reproduces the reference's
    traces exactly.  It never looks at the window."""

    def __init__(self, zoo: ModelZoo, b: Selector, correlation: float, rng: np.random.Generator):
        idx = b.indices()
        self.ids = [zoo.profiles[i].id for i in idx]
        self.mu = np.array([_positive_shift(zoo.profiles[i].target_auc) for i in idx])
        self.w_shared = math.sqrt(correlation)
        self.w_private = math.sqrt(1.0 - correlation)
        self.rng = rng

    def draw(self):
        y = 1.0 if self.rng.random() < 0.5 else 0.0
        shared = self.rng.standard_normal()
        private = self.rng.standard_normal(len(self.ids))
        s = self.mu * y + self.w_shared * shared + self.w_private * private
        return dict(zip(self.ids, map(float, s))), float(s.mean())


def check_modalities(zoo: ModelZoo, b: Selector, rates: dict) -> None:
    check_selector(b, zoo)
    if b.popcount == 0:
        raise EmptyEnsembleError("cannot serve an empty ensemble")
    missing = {zoo.profiles[i].modality for i in b.indices()} - set(rates)
    if missing:
        raise ConfigurationError(f"rates: no stream configured for modality {sorted(missing)[0]!r}")


class EngineScorer:
    """The per-tick predict call on the device, for `run_simulation(scorer=...)`.

    Owns an `EnsembleEngine` for `patients` beds; `source(start, count)`
    returns the next samples of every stream as [P, leads, count] float32
    (default: the seeded synthetic ECG of `synth.py`).  Each `tick()` appends
    one hop and scores every bed's latest window; it returns the host results
    and the measured device seconds of the tick graph.
    """

    def __init__(self, zoo: ModelZoo, b: Selector, patients: int, rates: dict, window_s: float, *,
                 hop: int | None = None, seed: int = 0, stream_seed: int = 0, device: int = 0, source=None):
        from .engine import EnsembleEngine
        check_modalities(zoo, b, rates)
        fs = set(float(r) for r in rates.values())
        if len(fs) != 1:
            raise ConfigurationError("rates: the device engine needs one common sampling rate for all leads")
        self.fs = fs.pop()
        self.window = samples_per_window("*", self.fs, window_s)
        leads = 1 + max(modality_lead(m) for m in rates)
        self.patients, self.leads = patients, leads
        self.hop = int(hop) if hop is not None else self.window
        if source is None:
            from . import synth

            def source(start, count, _p=patients, _l=leads):
                return synth.ecg_block(stream_seed, _p, _l, start, count)
        self.source = source
        self.engine = EnsembleEngine(zoo, b, patients, leads=leads, fs=int(round(self.fs)), window_s=window_s,
                                     hop=self.hop, seed=seed, device=device)
        self.pos = 0
        # the first window needs W samples: pre-ingest all but the first hop
        if self.window > self.hop:
            self.engine.ingest(self.source(0, self.window - self.hop))
            self.pos = self.window - self.hop

    def tick(self):
        block = self.source(self.pos, self.hop)
        res = self.engine.tick(block)
        self.pos += self.hop
        return res, self.engine.last_tick_seconds()

    def close(self):
        self.engine.close()


def run_simulation(zoo: ModelZoo, b: Selector, executor: ExecutorModel, patients: int, rates: dict,
                   window_s: float, duration_s: float, seed: int = 0, correlation: float = 0.5,
                   agg_overhead_s: float = DEFAULT_AGG_OVERHEAD_S, stagger: bool = False,
                   scorer: EngineScorer | None = None) -> list:
    """One QueryTrace per (patient, window); see the module docstring for the two scorers."""
    check_modalities(zoo, b, rates)
    if window_s <= 0 or duration_s < window_s:
        raise ConfigurationError("window_s must be positive and duration_s >= window_s")
    if patients < 1:
        raise ConfigurationError("patients must be >= 1")
    for modality, rate in rates.items():
        samples_per_window(modality, rate, window_s)
    if scorer is not None:
        return _run_ticks(zoo, b, patients, window_s, duration_s, agg_overhead_s, stagger, scorer)

    rng = np.random.default_rng(seed)
    phase = rng.uniform(0.0, window_s, patients) if stagger else np.zeros(patients)
    draw = BinormalScorer(zoo, b, correlation, rng).draw
    s_q = service_time(b, zoo, executor)
    FLUSH, DONE = 0, 1
    heap: list = []
    seq = 0
    for p in range(patients):
        for k in range(1, int(math.floor((duration_s - phase[p]) / window_s + 1e-9)) + 1):
            heap.append((phase[p] + k * window_s, seq, FLUSH, p))
            seq += 1
    heapq.heapify(heap)
    fifo: deque = deque()
    idle = executor.n_slots
    out: list = []
    qid = 0
    while heap:
        now, _, kind, item = heapq.heappop(heap)
        if kind == FLUSH:
            scores, ens = draw()
            q = (qid, item, now - window_s, now + agg_overhead_s, scores, ens)
            qid += 1
            if idle > 0 and not fifo:
                idle -= 1
                heapq.heappush(heap, (q[3] + s_q, seq, DONE, (q, q[3])))
                seq += 1
            else:
                fifo.append(q)
        else:
            q, began = item
            idle += 1
            out.append(QueryTrace(q[0], q[1], q[2], q[3], began, now, q[4], q[5]))
            if fifo:
                nq = fifo.popleft()
                idle -= 1
                start = max(now, nq[3])
                heapq.heappush(heap, (start + s_q, seq, DONE, (nq, start)))
                seq += 1
    out.sort(key=lambda t: t.query_id)
    return out


def _run_ticks(zoo, b, patients, window_s, duration_s, agg_overhead_s, stagger, scorer: EngineScorer) -> list:
    """Aligned device ticks: every hop all beds' latest windows are scored in one tick."""
    if stagger:
        raise ConfigurationError("stagger: the device engine serves aligned windows (one tick per hop)")
    if scorer.patients != patients:
        raise ConfigurationError(f"patients: scorer serves {scorer.patients} beds, simulation asks for {patients}")
    hop_s = scorer.hop / scorer.fs
    n_ticks = int(math.floor((duration_s - window_s) / hop_s + 1e-9)) + 1
    out = []
    gpu_free = 0.0
    qid = 0
    for k in range(n_ticks):
        t_flush = window_s + k * hop_s
        res, dev_s = scorer.tick()
        t_enq = t_flush + agg_overhead_s
        start = max(t_enq, gpu_free)
        done = start + dev_s
        gpu_free = done
        for p in range(patients):
            scores = dict(zip(res.member_ids, map(float, res.member_logits[p])))
            out.append(QueryTrace(qid, p, t_flush - window_s, t_enq, start, done, scores,
                                  float(res.ens_mean_logit[p])))
            qid += 1
    return out


def run_simulation_wallclock(zoo: ModelZoo, b: Selector, executor: ExecutorModel, patients: int, rates: dict,
                             window_s: float, duration_s: float, seed: int = 0, correlation: float = 0.5, *,
                             hop: int | None = None, device: int = 0, speedup: float = 1.0, source=None) -> list:
    """Wall-clock mode with the reference's signature (`runtime.py:321-396`), served by the device.

    The reference runs one ingest thread per patient feeding per-sample
    `Aggregator`s, emits a query when every needed modality flushed window k,
    and lets `executor.n_slots` workers `sleep(service_time)`.  Here a sensor
    thread delivers one frame per hop (every bed's and lead's newest samples,
    tumbling windows by default: hop = rate * window_s, exactly the
    Aggregator's windows) and one device worker scores each frame in ONE
    `EnsembleEngine.tick` (`serving.ServingLoop`).  The trace schema, ordering
    (query id = tick * patients + bed) and timestamps (seconds since start;
    `t_ingest` = the window's start) follow the reference.  `model_scores` are
    the members' real logits and `ensemble_score` the mean latent
    (`runtime.py:136`), not binormal draws, so `correlation` is accepted for
    signature compatibility only; the measured tick replaces `service_time`,
    so `executor` only validates.  `seed` seeds the synthetic ECG streams
    (`source(start, count) -> [P, leads, count]` overrides them; the
    reference's own generator sends 0.0, `synth.zero_stream`).  `speedup`
    compresses time (1.0 = real time, as the reference).
    """
    from . import synth
    from .engine import EnsembleEngine
    from .serving import ServingLoop
    check_modalities(zoo, b, rates)
    if not isinstance(executor, ExecutorModel):
        raise ConfigurationError("executor must be an ExecutorModel")
    if window_s <= 0 or duration_s < window_s:
        raise ConfigurationError("window_s must be positive and duration_s >= window_s")
    if patients < 1:
        raise ConfigurationError("patients must be >= 1")
    for modality, rate in rates.items():
        samples_per_window(modality, rate, window_s)
    fs = set(float(r) for r in rates.values())
    if len(fs) != 1:
        raise ConfigurationError("rates: the device engine needs one common sampling rate for all leads")
    fs_v = fs.pop()
    W = samples_per_window("*", fs_v, window_s)
    hop = W if hop is None else int(hop)
    leads = 1 + max(modality_lead(m) for m in rates)
    if source is None:
        def source(start, count, _p=patients, _l=leads):
            return synth.ecg_block(seed, _p, _l, start, count)
    # ticks whose window ends by duration_s (the reference flushes floor(duration * rate) samples)
    n_ticks = (int(math.floor(duration_s * fs_v + 1e-9)) - W) // hop + 1
    with EnsembleEngine(zoo, b, patients, leads=leads, fs=int(round(fs_v)), window_s=window_s, hop=hop,
                        seed=0, device=device) as eng:
        traces = ServingLoop(eng, source, speedup=speedup).run(n_ticks)
    return sorted(traces, key=lambda t: t.query_id)


def e2e_percentiles(traces: list) -> dict:
    """Nearest-rank p50/p95/p99 of done - enqueue ("query") and done - ingest ("capture")."""
    if not traces:
        raise ValueError("need at least one trace")

    def pct(vals):
        s = sorted(vals)
        n = len(s)
        return {f"p{q}": s[math.ceil(q / 100 * n) - 1] for q in (50, 95, 99)}

    return {"query": pct([t.t_done - t.t_enqueue for t in traces]),
            "capture": pct([t.t_done - t.t_ingest for t in traces])}


def queueing_delays(traces: list) -> list:
    return [t.t_dequeue - t.t_enqueue for t in traces]


def save_traces_jsonl(traces: list, path) -> None:
    """One JSON object per trace, keys sorted (runtime.py:259-264)."""
    with open(path, "w", encoding="utf-8") as fh:
        fh.writelines(json.dumps(asdict(t), sort_keys=True) + "\n" for t in traces)


@dataclass(frozen=True)
class TimelinePoint:
    t_s: float
    latency_s: float
    kind: str    # "aggregation" or "inference"


def batch_comparison(zoo: ModelZoo, b: Selector, executor: ExecutorModel, patients: int, rates: dict,
                     window_s: float, batch_period_s: float, duration_s: float, seed: int = 0,
                     agg_overhead_s: float = DEFAULT_AGG_OVERHEAD_S) -> tuple[list, list]:
    """Online per-window serving vs deferred batch processing (runtime.py:273-311), host only.

    Both timelines come from the parity-mode DES of the same seeded windows: online = one
    inference point per query (done - enqueue at its enqueue time); batch = at every period
    boundary the queries enqueued in that period drained back to back through the slots;
    plus one aggregation-only point per simulated second on both."""
    if batch_period_s < window_s:
        raise ConfigurationError("batch_period_s must be >= window_s")
    traces = run_simulation(zoo, b, executor, patients, rates, window_s, duration_s, seed=seed,
                            agg_overhead_s=agg_overhead_s)
    s_q = service_time(b, zoo, executor)
    online = [TimelinePoint(t.t_enqueue, t.t_done - t.t_enqueue, "inference") for t in traces]
    batch = []
    for m in range(1, int(math.floor(duration_s / batch_period_s + 1e-9)) + 1):
        hi = m * batch_period_s
        n = sum(1 for t in traces if hi - batch_period_s < t.t_enqueue - agg_overhead_s <= hi)
        if n:
            batch.append(TimelinePoint(hi, agg_overhead_s + math.ceil(n / executor.n_slots) * s_q, "inference"))
    for sec in range(int(duration_s)):
        online.append(TimelinePoint(float(sec), agg_overhead_s, "aggregation"))
        batch.append(TimelinePoint(float(sec), agg_overhead_s, "aggregation"))
    key = lambda pt: (pt.t_s, pt.kind)  # noqa: E731
    return sorted(online, key=key), sorted(batch, key=key)


def save_timeline_csv(points: list, path) -> None:
    """t_s,latency_s,kind rows with repr() floats (runtime.py:314-318)."""
    with open(path, "w", encoding="utf-8") as fh:
        fh.write("t_s,latency_s,kind\n")
        fh.writelines(f"{p.t_s!r},{p.latency_s!r},{p.kind}\n" for p in points)
