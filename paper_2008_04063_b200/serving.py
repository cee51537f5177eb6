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
import socket
import socketserver
import struct
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
        eng.prepare()  # graphs built and uploaded before the clock starts
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


# ---------------------------------------------------------------- binary ingest
# The reference's ingest adapter is newline-delimited JSON, one SensorSample
# per line (`IngestServer`, runtime.py:399-469): ~0.3 kB of text per sample.
# The device path consumes whole frames instead: every bed's and lead's newest
# `hop` samples as little-endian float32 [P, leads, hop] behind a 20-byte
# header, received straight into a pinned staging buffer and ticked.
FRAME_MAGIC = b"HBF1"
_HDR = struct.Struct("<4sIIII")   # magic, tick, patients, leads, hop


def encode_frame(tick: int, frame: np.ndarray) -> bytes:
    a = np.ascontiguousarray(frame, dtype="<f4")
    if a.ndim != 3:
        raise ValueError("frame must be [patients, leads, hop]")
    return _HDR.pack(FRAME_MAGIC, tick, *a.shape) + a.tobytes()


def send_frames(address, frames, first_tick: int = 0) -> None:
    """Client helper: push [P, leads, hop] frames to a BinaryIngestServer."""
    with socket.create_connection(address) as sock:
        for k, f in enumerate(frames):
            sock.sendall(encode_frame(first_tick + k, f))


def _recv_exact(rfile, n: int, out: memoryview | None = None):
    if out is None:
        data = rfile.read(n)
        return data if data is not None and len(data) == n else None
    got = 0
    while got < n:
        k = rfile.readinto(out[got:n])
        if not k:
            return None
        got += k
    return out


class BinaryIngestServer:
    """TCP server: binary frames -> one device tick each -> on_result(tick, TickResult).

    Frames of one connection are ticked in arrival order; a lock serialises
    ticks across connections (a context is single-threaded, as the reference
    serialises its scorer, runtime.py:367-368).  A malformed frame closes its
    connection and is recorded in `errors`.
    """

    def __init__(self, engine, on_result=None, host: str = "127.0.0.1", port: int = 0):
        self.engine = engine
        self.on_result = on_result
        self.errors: list = []
        self.ticks = 0
        self._lock = threading.Lock()
        shape = (engine.patients, engine.leads, engine.hop)
        self._shape = shape
        self._nbytes = int(np.prod(shape)) * 4
        try:  # pinned host staging so the H2D copy inside hb_tick is a DMA
            import torch
            self._pinned = torch.empty(shape, dtype=torch.float32, pin_memory=True).numpy()
        except Exception:  # noqa: BLE001 - no CUDA here: plain memory still works for framing
            self._pinned = np.empty(shape, np.float32)
        outer = self

        class Handler(socketserver.StreamRequestHandler):
            def handle(self):
                while True:
                    hdr = _recv_exact(self.rfile, _HDR.size)
                    if hdr is None:
                        return
                    magic, tick, P, leads, hop = _HDR.unpack(hdr)
                    if magic != FRAME_MAGIC or (P, leads, hop) != outer._shape:
                        outer.errors.append(f"bad frame header {magic!r} {(P, leads, hop)}")
                        return
                    with outer._lock:
                        buf = memoryview(outer._pinned.reshape(-1).view(np.uint8))
                        if _recv_exact(self.rfile, outer._nbytes, buf) is None:
                            outer.errors.append("truncated frame")
                            return
                        res = outer.engine.tick(outer._pinned)
                        outer.ticks += 1
                        if outer.on_result is not None:
                            outer.on_result(tick, res)

        self._server = socketserver.ThreadingTCPServer((host, port), Handler)
        self._server.daemon_threads = True
        self._thread = threading.Thread(target=self._server.serve_forever, daemon=True)

    @property
    def address(self):
        return self._server.server_address

    def start(self) -> None:
        self._thread.start()

    def stop(self) -> None:
        self._server.shutdown()
        self._server.server_close()
