"""The serving loop through the drop-in `run_simulation` with the device
scorer, `record_cohort`, and the measured latency profiler."""
import numpy as np
import pytest

from oracle import cpu_path, windows
from paper_2008_04063_b200 import cohort, composer, latency, runtime, synth
from paper_2008_04063_b200.zoo import Selector, holmes_zoo

pytestmark = pytest.mark.gpu
RATES = {"ECG-I": 250.0, "ECG-II": 250.0, "ECG-III": 250.0}


def test_run_simulation_with_engine_scorer_tumbling():
    """hop == window: query k of patient p scores reference window k; scores = real member logits."""
    zoo = holmes_zoo()
    sel = Selector.from_indices(60, [0, 21])
    P = 3
    sc = runtime.EngineScorer(zoo, sel, P, RATES, 30.0, stream_seed=4)
    try:
        tr = runtime.run_simulation(zoo, sel, latency.ExecutorModel(), P, RATES, 30.0, 90.0, scorer=sc)
    finally:
        sc.close()
    assert len(tr) == 3 * P
    streams = synth.ecg_block(4, P, 3, 0, 3 * 7500)
    for k in range(3):
        ml, _, mean_logit = cpu_path.cpu_tick(zoo, sel, streams, (k + 1) * 7500)
        for p in range(P):
            t = tr[k * P + p]
            assert t.patient_id == p and t.query_id == k * P + p
            assert t.t_ingest == 30.0 * k and t.t_enqueue == 30.0 * (k + 1) + 0.002
            assert t.t_done > t.t_dequeue >= t.t_enqueue
            got = np.array([t.model_scores[zoo.profiles[i].id] for i in sel.indices()])
            assert np.abs(got - ml[p]).max() <= 2e-2
            assert abs(t.ensemble_score - mean_logit[p]) <= 2e-2
    pc = runtime.e2e_percentiles(tr)
    assert 0 < pc["query"]["p99"] < 0.2        # well under the 200 ms SLO


def test_run_simulation_with_engine_scorer_sliding():
    zoo = holmes_zoo()
    sel = Selector.from_indices(60, [10])
    P = 2
    sc = runtime.EngineScorer(zoo, sel, P, RATES, 30.0, hop=250)
    try:
        tr = runtime.run_simulation(zoo, sel, latency.ExecutorModel(), P, RATES, 30.0, 33.0, scorer=sc)
    finally:
        sc.close()
    assert len(tr) == 4 * P                      # windows ending at 30, 31, 32, 33 s
    assert [t.t_ingest for t in tr[::P]] == [0.0, 1.0, 2.0, 3.0]
    with pytest.raises(runtime.ConfigurationError):
        sc2 = runtime.EngineScorer(zoo, sel, P, RATES, 30.0)
        try:
            runtime.run_simulation(zoo, sel, latency.ExecutorModel(), P, RATES, 30.0, 60.0, stagger=True, scorer=sc2)
        finally:
            sc2.close()


def test_record_cohort_then_sweep():
    """Member logits over recorded windows fill a Cohort; the sweep runs on it (config 4 shape, small)."""
    zoo = holmes_zoo()
    sel = Selector.from_indices(60, [0, 1, 20, 41])
    N = 40
    wins = np.stack([synth.ecg_block(11, [p], 3, 0, 7500)[0] for p in range(N)])
    labels = np.r_[np.ones(N // 2, np.int8), np.zeros(N - N // 2, np.int8)]
    coh = cohort.record_cohort(zoo, wins, labels, selector=sel, batch=16)
    assert coh.scores.shape == (N, 4)
    for j, i in enumerate(sel.indices()):
        prof = zoo.profiles[i]
        from oracle import cnn
        x = cnn.znorm(np.stack([windows.sliding_window(wins[r, prof.lead], 7500, 7500) for r in range(N)]))
        ref = cnn.member_forward(x, cpu_path.params_for(prof), prof.width, prof.depth)
        assert np.abs(coh.scores[:, j] - ref).max() <= 2e-2
    aucs = composer.sweep_aucs(coh)
    assert aucs.shape == (15,) and np.all((aucs >= 0) & (aucs <= 1))


def test_measured_latency_profiler():
    zoo = holmes_zoo()
    sysc = latency.SystemConfig(n_slots=1, patients=16)
    mp = latency.MeasuredLatencyProfiler(zoo, sysc, reps=3)
    t1 = mp.tick_seconds(Selector.from_indices(60, [10]))
    t2 = mp.tick_seconds(Selector.from_indices(60, [10, 13]))
    assert 0 < t1 < t2 < 0.2
    rep = mp.report(Selector.from_indices(60, [10, 13]))
    assert rep.feasible and rep.total_s < 0.2


def test_serving_loop_realtime():
    """Wall-clock mode (runtime.py:321-396 counterpart): frames at 100x real time, one tick per hop."""
    from paper_2008_04063_b200.engine import EnsembleEngine
    from paper_2008_04063_b200.serving import ServingLoop, frames_from, tick_latency_percentiles
    zoo = holmes_zoo()
    sel = Selector.from_indices(60, [10, 13])
    P, hop, n_ticks = 8, 250, 12
    streams = synth.ecg_block(6, P, 3, 0, 7500 + hop * n_ticks)
    with EnsembleEngine(zoo, sel, P, hop=hop) as eng:
        loop = ServingLoop(eng, frames_from(streams), speedup=100.0)
        tr = loop.run(n_ticks)
    assert len(tr) == P * n_ticks
    assert [t.query_id for t in tr] == list(range(P * n_ticks))
    pc = tick_latency_percentiles(tr, P)
    assert pc["p99"] < 0.2
    ml, _, _ = cpu_path.cpu_tick(zoo, sel, streams, 7500 + hop * (n_ticks - 1))
    last = tr[-P:]
    got = np.array([[t.model_scores[zoo.profiles[i].id] for i in sel.indices()] for t in last])
    assert np.abs(got - ml).max() <= 2e-2


def test_binary_ingest_server_ticks_match_direct_engine():
    from paper_2008_04063_b200.engine import EnsembleEngine
    from paper_2008_04063_b200.serving import BinaryIngestServer, send_frames
    import time
    zoo = holmes_zoo()
    sel = Selector.from_indices(60, [10, 13])
    P, hop = 4, 250
    streams = synth.ecg_block(8, P, 3, 0, 7500 + 3 * hop)
    frames = [streams[:, :, 7500 + k * hop - hop:7500 + k * hop] for k in range(4)]
    got = []
    with EnsembleEngine(zoo, sel, P, hop=hop) as eng:
        eng.ingest(streams[:, :, :7500 - hop])
        srv = BinaryIngestServer(eng, on_result=lambda k, r: got.append((k, r.ens_prob.copy())))
        srv.start()
        try:
            send_frames(srv.address, frames)
            t0 = time.time()
            while len(got) < 4 and time.time() - t0 < 30:
                time.sleep(0.01)
        finally:
            srv.stop()
    assert [k for k, _ in got] == [0, 1, 2, 3] and srv.errors == []
    with EnsembleEngine(zoo, sel, P, hop=hop) as ref:
        ref.ingest(streams[:, :, :7500 - hop])
        for k, f in enumerate(frames):
            assert np.array_equal(ref.tick(f).ens_prob, got[k][1])


@pytest.mark.parametrize("patients,jitter", [(16, 2.5e-4), (200, 2.5e-4), (8192, 2.5e-4), (3, 0.0)])
def test_device_arrival_curve_bit_identical(patients, jitter):
    """K7 vs the host formulation (= the reference's numpy loops): exact path
    (<= 8000 events) and binned path (8192 beds -> 16384 events, ~30 000 bins)."""
    sysc = latency.SystemConfig(patients=patients)
    tr = latency.profiling_trace(sysc, seed=1, jitter_s=jitter)
    a = latency.build_arrival_curve(tr, backend="host")
    b = latency.build_arrival_curve(tr, backend="device")
    assert np.array_equal(a.dts, b.dts) and np.array_equal(a.counts, b.counts)
    assert a.n_events == b.n_events and a.span_s == b.span_s
