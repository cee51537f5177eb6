"""K6 profiler sweep on the device vs the reference's own results (golden) and
the CPU oracle.  Bar: bit-exact AUCs and the identical selected ensemble."""
import os

import numpy as np
import pytest

from oracle import auc as oauc
from paper_2008_04063_b200 import cohort, composer, errors, latency, metrics, zoo

pytestmark = pytest.mark.gpu
G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def c4():
    z10 = zoo.load_zoo(os.path.join(G, "zoo_10.json"))
    return z10, cohort.synthesize_cohort(z10, 10000, 10000, 0.5, 0)


def test_sweep_matches_reference_exhaustive_search_bit_exact(c4):
    z10, coh = c4
    gold = np.load(os.path.join(G, "sweep_n10.npz"))
    aucs = composer.sweep_aucs(coh)
    assert aucs.shape == (1023,)
    assert np.array_equal(aucs, gold["auc"]), np.flatnonzero(aucs != gold["auc"])[:10]


def test_exhaustive_search_selects_the_reference_ensemble(c4):
    import json
    z10, coh = c4
    ref = json.load(open(os.path.join(G, "sweep_n10.json")))
    gold = np.load(os.path.join(G, "sweep_n10.npz"))
    lat = {v + 1: float(x) for v, x in enumerate(gold["latency"])}
    lp = lambda b: lat[b.as_int()]  # noqa: E731 - the reference LatencyProfiler's values
    res = composer.exhaustive_search(z10, coh, lp, budget_s=ref["budget_s"])
    assert str(res.best) == ref["best"] == "0000000111"
    assert res.best_objective == ref["best_objective"] and res.best_accuracy == ref["best_accuracy"]
    dual = composer.exhaustive_search(z10, coh, lp, budget_s=ref["budget_s"], accuracy_floor=ref["dual_floor"])
    assert str(dual.best) == ref["dual_best"] and dual.best_objective == ref["dual_objective"]
    # and with our own (host) LatencyProfiler restatement
    res2 = composer.exhaustive_search(z10, coh, latency.LatencyProfiler(z10, latency.ExecutorModel(),
                                                                        latency.SystemConfig()), budget_s=0.2)
    assert str(res2.best) == ref["best"]


def test_tie_heavy_cohort_bit_exact():
    t = np.load(os.path.join(G, "sweep_ties.npz"))
    coh = cohort.Cohort(labels=t["labels"], scores=t["scores"], seed=21)
    assert np.array_equal(composer.sweep_aucs(coh), t["auc"])


def test_metrics_golden_on_device():
    import json
    g = json.load(open(os.path.join(G, "metrics.json")))
    for case in g["known"]:
        assert metrics.roc_auc(case["labels"], case["scores"]) == case["roc_auc"]
    m = g["many"]
    got = metrics.roc_auc_many(np.array(m["labels"]), np.array(m["matrix"]))
    assert np.array_equal(got, np.array(m["auc"]))


def test_ensemble_scores_and_accuracy_profile(c4):
    import json
    z10, coh = c4
    g = json.load(open(os.path.join(G, "cohort.json")))
    small = cohort.synthesize_cohort(z10, 37, 50, 0.3, 4)
    for e in g["ensemble"]:
        b = zoo.Selector.from_indices(10, e["selected"])
        ens = cohort.ensemble_scores(coh, b)
        import hashlib
        assert hashlib.sha256(ens.tobytes()).hexdigest() == e["sha256_scores"]
        assert cohort.ensemble_roc_auc(coh, b) == e["roc_auc"]
        rep = cohort.accuracy_profile(small, b)
        assert [rep.roc_auc, rep.pr_auc, rep.f1, rep.accuracy] == e["report"]


@pytest.mark.parametrize("N,npos,n,seed", [(1, 1, 1, 0), (2, 1, 3, 1), (37, 5, 4, 2), (5000, 4999, 3, 3),
                                           (40000, 17000, 5, 4), (70000, 35000, 2, 5)])
def test_sweep_matches_oracle_on_edge_shapes(N, npos, n, seed):
    """Tiny / single-sample-class / heavily unbalanced / global-scratch (m > 16384) cohorts."""
    if N == 1:
        with pytest.raises(errors.UndefinedMetricError):
            cohort.DeviceCohort(np.zeros((1, 1)), np.array([1], np.int8))
        return
    rng = np.random.default_rng(seed)
    lab = np.zeros(N, np.int8)
    lab[rng.permutation(N)[:npos]] = 1
    sc = rng.standard_normal((N, n)) + 0.3 * lab[:, None]
    if seed % 2:
        sc = np.round(sc, 1)        # ties
    vals = np.arange(1, 1 << n)
    with cohort.DeviceCohort(sc, lab) as dc:
        got = dc.auc_range(1, len(vals))
    assert np.array_equal(got, oauc.sweep(lab, sc, vals))


def test_explicit_selectors_wide_zoo():
    """60-column cohort (the full zoo): explicit bit rows, the SMBO accuracy-profiler path."""
    z = zoo.holmes_zoo()
    coh = cohort.synthesize_cohort(z, 300, 500, 0.5, 9)
    rng = np.random.default_rng(1)
    bits = (rng.random((40, 60)) < 0.3).astype(np.uint8)
    bits[bits.sum(1) == 0, 0] = 1
    bits[0] = 1
    got = coh.device().auc_bits(bits)
    exp = np.array([oauc.roc_auc(coh.labels, oauc.ensemble_mean(coh.scores, np.flatnonzero(r))) for r in bits])
    assert np.array_equal(got, exp)
    f = composer.make_accuracy_profiler(coh)
    assert f(zoo.Selector(tuple(bits[3]))) == exp[3]


def test_sweep_errors():
    coh = cohort.Cohort(labels=np.array([0, 1, 1]), scores=np.zeros((3, 2)), seed=0)
    with pytest.raises(errors.EmptyEnsembleError):
        cohort.ensemble_roc_auc(coh, zoo.Selector.zeros(2))
    with pytest.raises(ValueError):
        cohort.ensemble_roc_auc(coh, zoo.Selector.ones(3))
    assert cohort.ensemble_roc_auc(coh, zoo.Selector.ones(2)) == 0.5   # all tied


def test_one_shot_hb_sweep_auc_matches_oracle_and_cohort_path(c4):
    """The one-shot C-ABI entry `hb_sweep_auc` (32-bit selector masks) gives the same AUCs as the
    persistent-cohort path and the CPU oracle, bit for bit."""
    z10, coh = c4
    masks = np.arange(1, 1024, 7, dtype=np.uint32)
    got = metrics.sweep_auc(coh.labels, coh.scores, masks)
    assert np.array_equal(got, oauc.sweep(coh.labels, coh.scores, masks.astype(np.int64)))
    assert np.array_equal(got, composer.sweep_aucs(coh)[masks - 1])


def test_n16_sweep_and_selection_match_reference_bit_exact():
    """c4 at n = 16: all 65 535 candidates' AUCs equal the reference's exhaustive_search
    (tests/golden/sweep_n16.npz, N = 20 000) bit for bit, and so does the selected ensemble with
    the reference's latency values."""
    z16 = zoo.generate_zoo(1, [8, 16, 32, 64], [2, 4, 8, 16], seed=3)
    coh = cohort.synthesize_cohort(z16, 10000, 10000, 0.5, 0)
    gold = np.load(os.path.join(G, "sweep_n16.npz"))
    aucs = composer.sweep_aucs(coh)
    assert aucs.shape == (65535,)
    bad = np.flatnonzero(aucs != gold["auc"])
    assert bad.size == 0, (bad[:10], aucs[bad[:3]], gold["auc"][bad[:3]])
    lat = gold["latency"]
    res = composer.exhaustive_search(z16, coh, lambda b: float(lat[b.as_int() - 1]), budget_s=0.2)
    assert res.best.as_int() == int(gold["best"][0])
    assert res.best_objective == float(gold["best_objective"][0])


def test_trajectory_csv_of_a_device_search_matches_reference_bytes(tmp_path):
    import json
    g = json.load(open(os.path.join(G, "helpers.json")))
    z10 = zoo.generate_zoo(1, [8, 16, 32, 64, 128], [2, 4], seed=3)
    c10 = cohort.synthesize_cohort(z10, 300, 300, 0.5, 0)
    res = composer.exhaustive_search(z10, c10, lambda s: 0.01 * sum(s.bits), budget_s=0.05)
    res.save_trajectory_csv(tmp_path / "t.csv")
    assert (tmp_path / "t.csv").read_text(encoding="utf-8") == g["trajectory_csv"]


def test_cohorts_wider_than_the_kernel_column_list():
    """The reference accepts any cohort width; a 300-column cohort is scored on device sub-cohorts
    of the selected columns, bit-exact against the oracle."""
    rng = np.random.default_rng(3)
    lab = (rng.random(3000) < 0.45).astype(np.int8)
    sc = rng.standard_normal((3000, 300)) + 0.3 * lab[:, None]
    coh = cohort.Cohort(labels=lab, scores=sc, seed=0)
    for cols in ([0], [5, 299], list(range(0, 300, 7)), [17, 18, 19, 250]):
        b = zoo.Selector.from_indices(300, cols)
        v = int(sum(1 << c for c in cols))
        assert cohort.ensemble_roc_auc(coh, b) == oauc.sweep(lab, sc, [v])[0]
        assert np.array_equal(cohort.ensemble_scores(coh, b), oauc.ensemble_mean(sc, cols))
