"""Binary frame ingest (§8f: replaces the ND-JSON IngestServer, runtime.py:399-469)
— framing, ordering and error handling with a host stand-in for the engine."""
import socket
import time

import numpy as np

from paper_2008_04063_b200 import serving


class FakeEngine:
    patients, leads, hop = 3, 3, 250

    def __init__(self):
        self.seen = []

    def tick(self, frame):
        self.seen.append(frame.copy())
        return float(frame.sum())


def _wait(pred, timeout=10.0):
    t0 = time.time()
    while not pred() and time.time() - t0 < timeout:
        time.sleep(0.01)
    return pred()


def test_frames_round_trip_in_order():
    eng = FakeEngine()
    got = []
    srv = serving.BinaryIngestServer(eng, on_result=lambda k, r: got.append((k, r)))
    srv.start()
    try:
        rng = np.random.default_rng(0)
        frames = [rng.standard_normal((3, 3, 250)).astype(np.float32) for _ in range(5)]
        serving.send_frames(srv.address, frames, first_tick=7)
        assert _wait(lambda: len(got) == 5)
        assert [k for k, _ in got] == [7, 8, 9, 10, 11]
        for f, s in zip(frames, eng.seen):
            assert np.array_equal(f, s)
        assert srv.errors == []
    finally:
        srv.stop()


def test_bad_header_and_truncation_are_rejected():
    eng = FakeEngine()
    srv = serving.BinaryIngestServer(eng)
    srv.start()
    try:
        with socket.create_connection(srv.address) as s:
            s.sendall(serving.encode_frame(0, np.zeros((2, 3, 250), np.float32)))   # wrong shape
        assert _wait(lambda: len(srv.errors) == 1)
        with socket.create_connection(srv.address) as s:
            s.sendall(serving.encode_frame(0, np.zeros((3, 3, 250), np.float32))[:100])  # truncated
        assert _wait(lambda: len(srv.errors) == 2)
        assert eng.seen == [] and "bad frame header" in srv.errors[0] and srv.errors[1] == "truncated frame"
    finally:
        srv.stop()


def test_wire_size_vs_ndjson():
    """One 1-s tick of 64 beds x 3 leads: binary frame vs the reference's ND-JSON lines."""
    import json
    f = np.zeros((64, 3, 250), np.float32)
    binary = len(serving.encode_frame(0, f))
    line = json.dumps({"modality": "ECG-II", "patient_id": 63, "t_gen": 12.344, "value": 0.123456789},
                      sort_keys=True) + "\n"
    assert binary == 20 + 64 * 3 * 250 * 4
    assert binary * 10 < len(line) * 64 * 3 * 250
