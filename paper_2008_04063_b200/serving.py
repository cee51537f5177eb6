"""Real-time serving loop: the device counterpart of the reference's
wall-clock mode (`pkg/src/zooserve/runtime.py:321-396`).

The reference runs one ingest thread per patient feeding per-sample
`Aggregator`s, an MPMC queue and `n_slots` worker threads that `sleep(s_q)`.
Here the sensor side delivers one frame per hop — every bed's and lead's
newest `hop` samples, `[P, leads, hop]` float32, the binary frame that
replaces the ND-JSON `SensorSample` lines (`runtime.py:399-469`) — into a
bounded queue; one device worker turns each frame into ONE tick
(`EnsembleEngine.tick`: H2D of the frame, ring append, window + z-norm, every
member, aggregate, D2H of the scores).  Trace timestamps are real wall-clock
seconds since start, in the reference's `QueryTrace` schema, one trace per
(bed, tick).  `speedup` compresses time for tests (hop/fs/speedup seconds
between frames).
"""

from __future__ import annotations

import queue
import threading
import time

import numpy as np

from .runtime import QueryTrace


class ServingLoop:
    def __init__(self, engine, source, *, speedup: float = 1.0, max_queue: int = 8):
        """engine: an EnsembleEngine; source(start, count) -> [P, leads, count] float32."""
        self.engine = engine
        self.source = source
        self.speedup = float(speedup)
        self.period = engine.hop / engine.fs / self.speedup
        self.window_s = engine.window / engine.fs / self.speedup
        self._q: queue.Queue = queue.Queue(maxsize=max_queue)
        self.dropped = 0

    def run(self, n_ticks: int, prefill: bool = True) -> list:
        eng = self.engine
        pos = 0
        if prefill and eng.window > eng.hop:
            eng.ingest(self.source(0, eng.window - eng.hop))
            pos = eng.window - eng.hop
        traces: list = []
        t0 = time.monotonic()
        frames = [self.source(pos + k * eng.hop, eng.hop) for k in range(n_ticks)]  # the sensors' future data

        def sensors():
            for k in range(n_ticks):
                due = (k + 1) * self.period          # the frame's last sample exists at this time
                now = time.monotonic() - t0
                if now < due:
                    time.sleep(due - now)
                self._q.put((k, time.monotonic() - t0, frames[k]))
            self._q.put(None)

        def device_worker():
            qid = 0
            res = None
            while True:
                item = self._q.get()
                if item is None:
                    return
                k, t_enq, frame = item
                t_deq = time.monotonic() - t0
                res = eng.tick(frame, out=res)
                t_done = time.monotonic() - t0
                t_ing = max(0.0, (k + 1) * self.period - self.window_s)
                for p in range(eng.patients):
                    scores = dict(zip(res.member_ids, map(float, res.member_logits[p])))
                    traces.append(QueryTrace(qid, p, min(t_ing, t_enq), t_enq, max(t_deq, t_enq),
                                             max(t_done, t_deq, t_enq), scores, float(res.ens_mean_logit[p])))
                    qid += 1

        th = [threading.Thread(target=sensors), threading.Thread(target=device_worker)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        return traces


def tick_latency_percentiles(traces: list, patients: int) -> dict:
    """Nearest-rank p50/p95/p99 of per-tick (done - enqueue), one sample per tick."""
    import math
    lat = sorted(traces[i].t_done - traces[i].t_enqueue for i in range(0, len(traces), patients))
    n = len(lat)
    return {f"p{q}": lat[math.ceil(q / 100 * n) - 1] for q in (50, 95, 99)} if n else {}


def frames_from(streams: np.ndarray):
    """source() over a preloaded [P, leads, n] array."""
    def source(start, count):
        return np.ascontiguousarray(streams[:, :, start:start + count])
    return source
