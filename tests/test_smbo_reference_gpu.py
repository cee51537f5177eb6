"""INTEGRATION.md §2 end to end: the reference's own `smbo_search`
(`pkg/src/zooserve/composer.py:496-521`, run unmodified from the installed copy in
baseline/_ref — never from /root/reference) driven by this package's device profilers:
a cohort recorded on the serving kernels (`cohort.record_cohort`), the device
accuracy profiler (`composer.make_accuracy_profiler`, K6) swapped in for
`zooserve.composer.make_accuracy_profiler` exactly as the recipe does, and the
measured latency profiler (`latency.MeasuredLatencyProfiler`, real grouped ticks)
as f_l under the paper's 200 ms budget.  Skipped when baseline/_ref is absent."""
import os
import sys

import numpy as np
import pytest

from oracle import auc as oauc
from paper_2008_04063_b200 import cohort as hc
from paper_2008_04063_b200 import composer as hcomp
from paper_2008_04063_b200 import latency as hl
from paper_2008_04063_b200 import synth
from paper_2008_04063_b200.zoo import holmes_zoo

pytestmark = pytest.mark.gpu
REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")


def _zooserve():
    if not os.path.isdir(os.path.join(REF, "zooserve")):
        pytest.skip("the reference is not installed in baseline/_ref")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import zooserve.cohort as zcoh
    import zooserve.composer as zc
    import zooserve.zoo as zz
    return zc, zcoh, zz


def test_reference_smbo_with_device_profilers(monkeypatch):
    zc, zcoh, zz = _zooserve()
    z = holmes_zoo()
    rz = zz.generate_zoo(3, [8, 16, 32, 64, 128], [2, 4, 8, 16], 1)   # the reference's own 60-member zoo
    assert [p.id for p in rz.profiles] == [p.id for p in z.profiles]
    N, W = 384, 7500
    windows = synth.ecg_block(11, N, 3, 0, W)
    labels = (np.arange(N) % 3 == 0).astype(np.int8)
    windows[labels == 1] *= 1.5                                      # a class-dependent amplitude
    coh = hc.record_cohort(z, windows, labels, batch=128)            # member logits on the serving kernels
    monkeypatch.setattr(zc, "make_accuracy_profiler", lambda c: hcomp.make_accuracy_profiler(coh))
    lat = hl.MeasuredLatencyProfiler(z, hl.SystemConfig(patients=16), reps=3)
    try:
        params = zc.SearchParams(n_warm=5, n_iters=2, n_explore=40, top_k=3, seed=0)
        ref_cohort = zcoh.Cohort(labels=coh.labels, scores=coh.scores, seed=0)
        res = zc.smbo_search(rz, ref_cohort, lat, budget_s=0.2, params=params)
        assert res.feasible and res.best_latency_s <= 0.2
        assert res.profiler_calls <= params.n_warm + params.n_iters * params.top_k
        # the search's accuracy is the device AUC, which is the exact midrank AUC of the ensemble mean
        sel = np.array(res.best.bits, dtype=np.uint8)
        assert res.best_accuracy == hcomp.make_accuracy_profiler(coh)(res.best)
        exp = oauc.sweep(coh.labels, coh.scores, [int(sum(int(b) << k for k, b in enumerate(sel)))])[0]
        assert res.best_accuracy == exp
        assert res.best_latency_s == lat(res.best)
    finally:
        lat.close()
