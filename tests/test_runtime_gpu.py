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
    """The measured f_l times the candidate's real grouped tick: a 3-member ensemble of one
    architecture costs far less than three separate ticks (grouped into one launch per layer),
    measurements are cached per architecture multiset (leads do not matter), and mode="sum"
    (the cheap additive estimate) is an upper bound."""
    zoo = holmes_zoo()
    sysc = latency.SystemConfig(n_slots=1, patients=16)
    mp = latency.MeasuredLatencyProfiler(zoo, sysc, reps=3)
    try:
        t1 = mp.tick_seconds(Selector.from_indices(60, [10]))
        t2 = mp.tick_seconds(Selector.from_indices(60, [10, 13]))
        t3 = mp.tick_seconds(Selector.from_indices(60, [10, 30, 50]))      # three w32-d8, one per lead
        assert 0 < t1 < t2 < 0.2 and t1 < t3 < 2.5 * t1
        n = mp.measurements()
        assert mp.tick_seconds(Selector.from_indices(60, [30])) == t1     # same architecture, other lead
        assert mp.measurements() == n
        rep = mp.report(Selector.from_indices(60, [10, 13]))
        assert rep.feasible and rep.total_s < 0.2
    finally:
        mp.close()
    ms = latency.MeasuredLatencyProfiler(zoo, sysc, reps=3, mode="sum")
    try:
        assert ms.tick_seconds(Selector.from_indices(60, [10, 30, 50])) >= 0.9 * t3
    finally:
        ms.close()


def test_exhaustive_search_with_measured_latency_profiler():
    """SURVEY §8f row 1 end to end: composer.exhaustive_search over the n = 10 c4 cohort with the
    device-measured f_l (every candidate's real tick at 64 beds) picks a feasible ensemble under
    the paper's 200 ms budget, and its objective matches a re-evaluation of that selector."""
    import os
    from paper_2008_04063_b200 import zoo as hz
    z10 = hz.load_zoo(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "zoo_10.json"))
    coh = cohort.synthesize_cohort(z10, 2000, 2000, 0.5, 0)
    sysc = latency.SystemConfig(n_slots=1, patients=64)
    mp = latency.MeasuredLatencyProfiler(z10, sysc, reps=3)
    try:
        res = composer.exhaustive_search(z10, coh, mp, budget_s=0.2)
        assert res.feasible and res.best_latency_s < 0.2
        assert res.best_accuracy == composer.make_accuracy_profiler(coh)(res.best)
        assert mp.measurements() <= 1023
    finally:
        mp.close()


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


@pytest.mark.parametrize("beds", [16, 1024, 4100, 8192])
def test_device_arrival_curve_matches_reference_golden(beds):
    """K7 against the REFERENCE's own curves (tests/golden/curves.npz, make_golden.py): the exact
    branch and the binned branch (4100 beds = 8200 events, 8192 beds = 16 384 events)."""
    import os
    g = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "curves.npz"))
    ts = latency.profiling_trace(latency.SystemConfig(patients=beds), seed=7)
    a = latency.build_arrival_curve(ts, backend="device")
    assert np.array_equal(a.dts, g[f"b{beds}_dts"]) and np.array_equal(a.counts, g[f"b{beds}_counts"])


def test_run_simulation_wallclock_drop_in_signature():
    """`run_simulation_wallclock(zoo, b, executor, patients, rates, window_s, duration_s, seed,
    correlation)` with the reference's signature (runtime.py:321-396): one trace per (bed, window),
    tumbling windows (= the reference Aggregator's), ordered timestamps, query ids in (window, bed)
    order, and scores = the members' real logits on window k (oracle-checked).  Time runs 30x."""
    zoo = holmes_zoo()
    sel = Selector.from_indices(60, [10, 30])          # leads I and II
    P, speed, seed = 4, 30.0, 3
    ex = latency.ExecutorModel(n_slots=2)
    tr = runtime.run_simulation_wallclock(zoo, sel, ex, P, RATES, 30.0, 90.0, seed, 0.5, speedup=speed)
    assert len(tr) == 3 * P and [t.query_id for t in tr] == list(range(3 * P))
    for t in tr:
        assert t.t_ingest <= t.t_enqueue <= t.t_dequeue <= t.t_done
        assert set(t.model_scores) == {"ecg-i-w32-d8", "ecg-ii-w32-d8"}
    assert [round(tr[k * P].t_ingest * speed, 6) for k in range(3)] == [0.0, 30.0, 60.0]
    streams = synth.ecg_block(seed, P, 3, 0, 3 * 7500)
    for k in range(3):
        ml, _, mlog = cpu_path.cpu_tick(zoo, sel, streams, (k + 1) * 7500)
        got = np.array([[tr[k * P + p].model_scores[zoo.profiles[i].id] for i in sel.indices()] for p in range(P)])
        assert np.abs(got - ml).max() <= 2e-2
        assert np.abs(np.array([tr[k * P + p].ensemble_score for p in range(P)]) - mlog).max() <= 2e-2
    pc = runtime.e2e_percentiles(tr)
    assert pc["query"]["p99"] < 0.2
    with pytest.raises(runtime.ConfigurationError):
        runtime.run_simulation_wallclock(zoo, sel, ex, P, {"ECG-I": 250.0}, 30.0, 90.0)
