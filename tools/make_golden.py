#!/usr/bin/env python
"""Generate tests/golden/* by running the REFERENCE (zooserve, read-only at
/root/reference/pkg/src) in this container.

The fixtures pin the oracle and the host-side drop-in API against the
reference's own outputs on the same seeded inputs; the GPU box never reads
/root/reference (it only reads these committed files).  Re-run with
`python tools/make_golden.py` after changing a case; the script is
deterministic (numpy PCG64 streams, no wall clock).

Fixtures:
  seeds.json        derive_seed on assorted keys                    (seeds.py:15-19)
  zoo_60.json       generate_zoo(3, [8..128], [2,4,8,16], seed=1)    (zoo.py:150-195)
  zoo_10.json       generate_zoo(1, [8..128], [2,4], seed=3)         (c4 sweep zoo)
  windows.json      Aggregator windows of synthetic streams          (runtime.py:76-115)
  traces.json       run_simulation traces + e2e_percentiles          (runtime.py:153-251)
  metrics.json      roc_auc / roc_auc_many known answers + ties      (metrics.py:30-76)
  cohort.json       positive_shift, synthesize_cohort digests,
                    ensemble_scores / accuracy_profile               (cohort.py:27-115)
  sweep_n10.npz     exhaustive_search over the c4 cohort: every selector's AUC,
                    latency and the selected ensemble                 (composer.py:597-638)
  sweep_ties.npz    exhaustive_search AUCs on a tie-heavy cohort (n=8)
  latency.json      service_time / measure_capacity / LatencyProfiler (latency.py:145-333)
  curves.npz        build_arrival_curve on profiling traces of 16..8192 beds: the exact
                    branch and the binned branch above 8000 events (latency.py:198-239)
  sweep_n16.npz     exhaustive_search at n = 16 (65 535 candidates, N = 20 000)
  helpers.json      save_traces_jsonl, batch_comparison + save_timeline_csv, save_cohort_csv,
                    SearchResult.save_trajectory_csv, curves_to_csv, r2, constraint_penalty(nan)
"""
from __future__ import annotations

import hashlib
import json
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/pkg/src"
OUT = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)
sys.path.insert(0, REF)

from zooserve import cohort as rc  # noqa: E402
from zooserve import composer as rcomp  # noqa: E402
from zooserve import latency as rl  # noqa: E402
from zooserve import metrics as rm  # noqa: E402
from zooserve import runtime as rr  # noqa: E402
from zooserve import seeds as rs  # noqa: E402
from zooserve import zoo as rz  # noqa: E402

from paper_2008_04063_b200 import synth  # noqa: E402  (stream generator only)


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def dump(name, obj):
    with open(os.path.join(OUT, name), "w", encoding="utf-8") as fh:
        json.dump(obj, fh, indent=1, sort_keys=True)
        fh.write("\n")


def gen_seeds():
    keys = [(0,), (0, "warm"), (7, "ecg", 3, 1, 12), (1, "weights", "ecg-i-w32-d8"), ("x", 1.5, None),
            (12345, "baseline-rd")]
    dump("seeds.json", [{"key": list(map(repr, k)), "repr_key": "/".join(repr(x) for x in k),
                         "seed": rs.derive_seed(*k)} for k in keys])


def gen_zoos():
    rz.save_zoo(rz.generate_zoo(3, [8, 16, 32, 64, 128], [2, 4, 8, 16], seed=1), os.path.join(OUT, "zoo_60.json"))
    rz.save_zoo(rz.generate_zoo(1, [8, 16, 32, 64, 128], [2, 4], seed=3), os.path.join(OUT, "zoo_10.json"))


def gen_windows():
    """Feed the reference Aggregator sample by sample (SensorSample at t=(i+1)/rate,
    the wall-clock schedule of runtime.py:349-353) and record every window."""
    cases = []
    for (P, leads, rate, window_s, n_windows, seed) in [(2, 3, 250, 30.0, 2, 0), (3, 1, 10, 3.0, 4, 5),
                                                         (1, 2, 250, 2.0, 3, 9)]:
        W = int(round(rate * window_s))
        n = W * n_windows + W // 3  # trailing partial window never flushes
        out = []
        for p in range(P):
            for lead in range(leads):
                modality = rz._lead_modality(lead + 1)
                agg = rr.Aggregator(p, modality, rate, window_s)
                stream = synth.ecg_samples(seed, p, lead, 0, n, fs=rate)
                if p == P - 1 and lead == 0:
                    stream = np.zeros(n, np.float32)  # the reference wall-clock generator's signal
                for i, v in enumerate(stream):
                    b = agg.add(rr.SensorSample(p, modality, (i + 1) / rate, float(v)))
                    if b is not None:
                        out.append({"patient": p, "lead": lead, "modality": b.modality,
                                    "window_start_s": b.window_start_s, "t_flush": b.t_flush,
                                    "n": int(b.samples.size), "sha256_f64": sha(b.samples),
                                    "first": float(b.samples[0]), "last": float(b.samples[-1])})
        cases.append({"patients": P, "leads": leads, "rate": rate, "window_s": window_s, "seed": seed,
                      "n_samples": n, "zero_stream": [P - 1, 0], "windows": out})
    # out-of-order rejection and the rate*window validation
    errors = {}
    try:
        rr.Aggregator(0, "ECG-I", 250, 0.0021)
    except Exception as exc:  # noqa: BLE001
        errors["bad_rate_window"] = type(exc).__name__
    agg = rr.Aggregator(0, "ECG-I", 10, 1.0)
    agg.add(rr.SensorSample(0, "ECG-I", 1.0, 0.0))
    try:
        agg.add(rr.SensorSample(0, "ECG-I", 0.5, 0.0))
    except Exception as exc:  # noqa: BLE001
        errors["out_of_order"] = type(exc).__name__
    dump("windows.json", {"cases": cases, "errors": errors})


def _trace_dict(t):
    return {"query_id": t.query_id, "patient_id": t.patient_id, "t_ingest": t.t_ingest,
            "t_enqueue": t.t_enqueue, "t_dequeue": t.t_dequeue, "t_done": t.t_done,
            "model_scores": t.model_scores, "ensemble_score": t.ensemble_score}


def gen_traces():
    zoo = rz.generate_zoo(3, [8, 16, 32, 64, 128], [2, 4, 8, 16], seed=1)
    rates = {"ECG-I": 250.0, "ECG-II": 250.0, "ECG-III": 250.0}
    cases = []
    for (sel, P, dur, slots, stagger, seed) in [([10, 13, 30, 50], 4, 120.0, 2, False, 0),
                                                 ([10, 13, 30, 50], 5, 95.0, 1, True, 3),
                                                 ([0], 1, 60.0, 2, False, 0),
                                                 (list(range(60)), 6, 90.0, 2, False, 1)]:
        b = rz.Selector.from_indices(60, sel)
        ex = rl.ExecutorModel(n_slots=slots)
        tr = rr.run_simulation(zoo, b, ex, P, rates, 30.0, dur, seed=seed, stagger=stagger)
        cases.append({"selected": sel, "patients": P, "duration_s": dur, "n_slots": slots, "stagger": stagger,
                      "seed": seed, "service_time": rl.service_time(b, zoo, ex),
                      "traces": [_trace_dict(t) for t in tr], "percentiles": rr.e2e_percentiles(tr)})
    errs = {}
    for name, kw in [("empty", dict(b=rz.Selector.zeros(60))),
                     ("missing_modality", dict(rates={"ECG-I": 250.0}, b=rz.Selector.from_indices(60, [30]))),
                     ("short_duration", dict(duration_s=10.0)), ("no_patients", dict(patients=0))]:
        args = dict(zoo=zoo, b=rz.Selector.from_indices(60, [10]), executor=rl.ExecutorModel(), patients=2,
                    rates=rates, window_s=30.0, duration_s=60.0)
        args.update(kw)
        try:
            rr.run_simulation(**args)
            errs[name] = None
        except Exception as exc:  # noqa: BLE001
            errs[name] = [type(exc).__name__, str(exc)]
    dump("traces.json", {"cases": cases, "errors": errs})


def gen_metrics():
    known = []
    for labels, scores in [([0, 0, 1, 1], [.1, .2, .8, .9]), ([1, 1, 0, 0], [.1, .2, .8, .9]),
                           ([0, 1, 0, 1], [.1, .2, .3, .4]), ([0, 1, 0, 1], [.5, .5, .5, .5]),
                           ([1, 0, 1, 0, 1], [.3, .3, .7, .1, .3])]:
        known.append({"labels": labels, "scores": scores, "roc_auc": rm.roc_auc(labels, scores)})
    rng = np.random.default_rng(11)
    labels = (rng.random(501) < 0.37).astype(np.int8)
    mat = np.round(rng.standard_normal((501, 6)), 1)  # heavy ties
    mat[:, 5] = 0.25                                 # one all-tied column
    many = rm.roc_auc_many(labels, mat)
    errs = {}
    for name, (lab, sc) in {"single_class": ([1, 1, 1], [.1, .2, .3]), "bad_label": ([0, 2], [.1, .2]),
                            "nonfinite": ([0, 1], [0.1, float("nan")]), "empty": ([], []),
                            "shape": ([0, 1], [0.1])}.items():
        try:
            rm.roc_auc(lab, sc)
            errs[name] = None
        except Exception as exc:  # noqa: BLE001
            errs[name] = type(exc).__name__
    dump("metrics.json", {"known": known, "many": {"seed": 11, "labels": labels.tolist(), "matrix": mat.tolist(),
                                                   "auc": many.tolist()}, "errors": errs})


def gen_cohort():
    zoo10 = rz.generate_zoo(1, [8, 16, 32, 64, 128], [2, 4], seed=3)
    c = rc.synthesize_cohort(zoo10, 10000, 10000, correlation=0.5, seed=0)
    small = rc.synthesize_cohort(zoo10, 37, 50, correlation=0.3, seed=4)
    sels = [[0], [0, 1, 2], [9], list(range(10)), [3, 7]]
    out = {
        "positive_shift": {str(a): rc.positive_shift(a) for a in (0.5, 0.6, 0.75, 0.9, 0.99)},
        "c4": {"n_pos": 10000, "n_neg": 10000, "correlation": 0.5, "seed": 0,
               "sha256_scores": sha(c.scores), "sha256_labels": sha(c.labels)},
        "small": {"n_pos": 37, "n_neg": 50, "correlation": 0.3, "seed": 4, "sha256_scores": sha(small.scores),
                  "sha256_labels": sha(small.labels)},
        "ensemble": [{"selected": s, "sha256_scores": sha(rc.ensemble_scores(c, rz.Selector.from_indices(10, s))),
                      "roc_auc": rc.ensemble_roc_auc(c, rz.Selector.from_indices(10, s)),
                      "report": list(map(float, vars(rc.accuracy_profile(small, rz.Selector.from_indices(10, s)))
                                         .values()))}
                     for s in sels],
    }
    dump("cohort.json", out)


def gen_sweeps():
    zoo10 = rz.generate_zoo(1, [8, 16, 32, 64, 128], [2, 4], seed=3)
    c = rc.synthesize_cohort(zoo10, 10000, 10000, correlation=0.5, seed=0)
    sysc = rl.SystemConfig()
    lp = rl.LatencyProfiler(zoo10, rl.ExecutorModel(), sysc)
    res = rcomp.exhaustive_search(zoo10, c, lp, budget_s=sysc.budget_s, sys=sysc)
    aucs = np.array([r.accuracy for r in res.profiled])
    lats = np.array([r.latency_s for r in res.profiled])
    np.savez_compressed(os.path.join(OUT, "sweep_n10.npz"), auc=aucs, latency=lats,
                        best=np.array([int(res.best.as_int() if hasattr(res.best, "as_int") else
                                           sum(b << k for k, b in enumerate(res.best.bits)))]),
                        best_objective=np.array([res.best_objective]))
    # dual problem (latency minimisation under an accuracy floor)
    dual = rcomp.exhaustive_search(zoo10, c, lp, budget_s=sysc.budget_s, sys=sysc, accuracy_floor=0.9)
    with open(os.path.join(OUT, "sweep_n10.json"), "w") as fh:
        json.dump({"best": str(res.best), "best_objective": res.best_objective, "best_accuracy": res.best_accuracy,
                   "best_latency_s": res.best_latency_s, "dual_floor": 0.9, "dual_best": str(dual.best),
                   "dual_objective": dual.best_objective, "budget_s": sysc.budget_s}, fh, indent=1)
    # tie-heavy cohort: scores rounded to 0.5 -> many exact ties in every ensemble mean
    rng = np.random.default_rng(21)
    n, N = 8, 3000
    labels = np.concatenate([np.ones(1200, np.int8), np.zeros(N - 1200, np.int8)])
    scores = np.round(rng.standard_normal((N, n)) * 2 + labels[:, None] * 0.7) / 2
    tc = rc.Cohort(labels=labels, scores=scores, seed=21)
    zoo8 = rz.generate_zoo(1, [8, 16], [2, 4, 8, 16], seed=2)
    tres = rcomp.exhaustive_search(zoo8, tc, lambda b: 0.0, budget_s=1.0)
    np.savez_compressed(os.path.join(OUT, "sweep_ties.npz"), labels=labels, scores=scores,
                        auc=np.array([r.accuracy for r in tres.profiled]),
                        best=np.array([sum(b << k for k, b in enumerate(tres.best.bits))]))


def gen_latency():
    zoo = rz.generate_zoo(3, [8, 16, 32, 64, 128], [2, 4, 8, 16], seed=1)
    out = {"service_time": {}, "capacity": {}, "profiler": {}, "divergence": None}
    for name, idx in [("c1", [10]), ("c2", [10, 13, 30, 50]), ("w8d2", [0]), ("full", list(range(60)))]:
        b = rz.Selector.from_indices(60, idx)
        for slots in (1, 2, 8):
            ex = rl.ExecutorModel(n_slots=slots)
            out["service_time"][f"{name}/{slots}"] = rl.service_time(b, zoo, ex)
            out["capacity"][f"{name}/{slots}"] = rl.measure_capacity(b, zoo, ex)
    for name, idx, pts in [("c1", [10], 16), ("c2", [10, 13, 30, 50], 64), ("c2", [10, 13, 30, 50], 16)]:
        b = rz.Selector.from_indices(60, idx)
        sysc = rl.SystemConfig(n_slots=2, patients=pts)
        rep = rl.LatencyProfiler(zoo, rl.ExecutorModel(n_slots=2), sysc).report(b)
        out["profiler"][f"{name}/{pts}"] = [rep.serving_p95_s, rep.queue_bound_s, rep.total_s, rep.capacity_qps]
    try:
        sysc = rl.SystemConfig(n_slots=1, patients=100)
        rl.LatencyProfiler(zoo, rl.ExecutorModel(n_slots=1), sysc)(rz.Selector.ones(60))
    except Exception as exc:  # noqa: BLE001
        out["divergence"] = [type(exc).__name__, str(exc)]
    dump("latency.json", out)


def gen_curves():
    """The reference's build_arrival_curve on profiling traces of growing bed counts: exact branch
    (<= 8000 events) and the binned branch (latency.py:223-239) at 4100 and 8192 beds."""
    out = {}
    for beds in (16, 64, 1024, 4000, 4100, 8192):
        sysc = rl.SystemConfig(patients=beds)
        ts = rl.profiling_trace(sysc, seed=7)
        a = rl.build_arrival_curve(ts)
        out[f"b{beds}_dts"] = np.asarray(a.dts)
        out[f"b{beds}_counts"] = np.asarray(a.counts)
        out[f"b{beds}_meta"] = np.array([a.n_events, a.span_s])
    np.savez_compressed(os.path.join(OUT, "curves.npz"), **out)


def gen_sweep_n16():
    """exhaustive_search at n = 16 (65 535 candidates) over the c4-sized cohort (N = 20 000)."""
    zoo16 = rz.generate_zoo(1, [8, 16, 32, 64], [2, 4, 8, 16], seed=3)
    c = rc.synthesize_cohort(zoo16, 10000, 10000, correlation=0.5, seed=0)
    sysc = rl.SystemConfig()
    lp = rl.LatencyProfiler(zoo16, rl.ExecutorModel(), sysc)
    res = rcomp.exhaustive_search(zoo16, c, lp, budget_s=sysc.budget_s, sys=sysc)
    np.savez_compressed(os.path.join(OUT, "sweep_n16.npz"),
                        auc=np.array([r.accuracy for r in res.profiled]),
                        latency=np.array([r.latency_s for r in res.profiled]),
                        best=np.array([sum(b << k for k, b in enumerate(res.best.bits))]),
                        best_objective=np.array([res.best_objective]), best_accuracy=np.array([res.best_accuracy]),
                        scores_sha=np.array([sha(c.scores)]))


def gen_helpers():
    """The reference's host-side I/O helpers and small metrics, as file contents / values: traces
    JSONL, batch_comparison timelines CSV, cohort CSV, trajectory CSV, curves CSV, r2, and the hard
    constraint penalty on a NaN slack."""
    import tempfile
    out = {}
    zoo = rz.generate_zoo(3, [8, 16, 32, 64, 128], [2, 4, 8, 16], seed=1)
    b = rz.Selector.from_indices(60, [10, 13, 30, 50])
    rates = {"ECG-I": 250.0, "ECG-II": 250.0, "ECG-III": 250.0}
    ex = rl.ExecutorModel(n_slots=2)
    with tempfile.TemporaryDirectory() as d:
        def text(fn, *a):
            path = os.path.join(d, "f")
            fn(*a, path)
            return open(path, encoding="utf-8").read()
        tr = rr.run_simulation(zoo, b, ex, 3, rates, 30.0, 90.0, seed=4)
        out["traces_jsonl"] = text(rr.save_traces_jsonl, tr)
        on, ba = rr.batch_comparison(zoo, b, ex, 5, rates, 30.0, 120.0, 600.0, seed=2)
        out["timeline_online_csv"] = text(rr.save_timeline_csv, on)
        out["timeline_batch_csv"] = text(rr.save_timeline_csv, ba)
        c = rc.synthesize_cohort(rz.generate_zoo(1, [8, 16], [2], seed=3), 6, 5, correlation=0.5, seed=1)
        out["cohort_csv"] = text(rc.save_cohort_csv, c)
        zoo10 = rz.generate_zoo(1, [8, 16, 32, 64, 128], [2, 4], seed=3)
        c10 = rc.synthesize_cohort(zoo10, 300, 300, correlation=0.5, seed=0)
        res = rcomp.exhaustive_search(zoo10, c10, lambda s: 0.01 * sum(s.bits), budget_s=0.05)
        out["trajectory_csv"] = text(lambda p: res.save_trajectory_csv(p))
        ts = rl.profiling_trace(rl.SystemConfig(patients=16), seed=3)
        out["curves_csv"] = text(rl.curves_to_csv, rl.build_arrival_curve(ts),
                                 rl.ServiceCurve(rate_qps=5.0, latency_offset_s=0.01))
    rng = np.random.default_rng(8)
    a = rng.standard_normal(50)
    out["r2"] = [rm.r2(a + 0.1 * rng.standard_normal(50), a), rm.r2(a[::-1].copy(), a)]
    out["penalty_nan_slack"] = rcomp.constraint_penalty(float("nan"))
    dump("helpers.json", out)


def main():
    os.makedirs(OUT, exist_ok=True)
    if len(sys.argv) > 1:          # regenerate only the named fixtures, e.g. `make_golden.py curves sweep_n16`
        for name in sys.argv[1:]:
            globals()[f"gen_{name}"]()
        return
    gen_seeds()
    gen_zoos()
    gen_windows()
    gen_traces()
    gen_metrics()
    gen_cohort()
    gen_latency()
    gen_sweeps()
    gen_curves()
    gen_sweep_n16()
    gen_helpers()
    with open(os.path.join(OUT, "VERSIONS.json"), "w") as fh:
        import sklearn
        json.dump({"numpy": np.__version__, "sklearn": sklearn.__version__, "python": sys.version.split()[0],
                   "reference": REF}, fh, indent=1)
        fh.write("\n")
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
